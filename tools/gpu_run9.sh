set +e
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/pytest_gpu9.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu9.log
timeout 600 python tools/time_cases.py 1,4096,4096,2,2 16,4096,4096,2,2 16,11008,4096,4,4 16,4096,11008,4,4 1,11008,4096,1,2 2048,4096,4096,4,4 2048,11008,4096,2,8 > gpurun_out/dec9.log 2>&1
echo done >> gpurun_out/dec9.log
