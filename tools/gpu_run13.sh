set +e
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/pytest_gpu13.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu13.log
timeout 600 python tools/bench_kernels.py --suite decode --out gpurun_out/kernels13_decode.jsonl > gpurun_out/kernels13.log 2>&1
timeout 600 python tools/time_cases.py 2048,4096,4096,4,4 2048,11008,4096,2,8 2048,4096,11008,4,4 > gpurun_out/pre13.log 2>&1
timeout 300 python tools/tc_trace.py 2048 4096 4096 4 4 > gpurun_out/trace13.log 2>&1
