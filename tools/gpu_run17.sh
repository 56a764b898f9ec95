set +e
cd $GRAFT_REPO_ROOT
timeout 300 python tools/dbg_split.py > gpurun_out/dbg17.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/pytest_gpu17.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu17.log
timeout 300 python tools/tc_trace.py 16 4096 4096 2 2 > gpurun_out/trace17_dec.log 2>&1
timeout 300 python tools/time_cases.py 16,4096,4096,2,2 16,11008,4096,4,4 1,4096,4096,2,2 > gpurun_out/dec17.log 2>&1
