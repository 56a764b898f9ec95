set +e
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/pytest_gpu12.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu12.log
timeout 300 python tools/mma_trace.py 1,4096,4096,2,2 16,4096,4096,2,2 16,11008,4096,4,4 16,4096,11008,4,4 > gpurun_out/mtrace12.log 2>&1
timeout 600 python tools/bench_kernels.py --suite decode --out gpurun_out/kernels12_decode.jsonl > gpurun_out/kernels12.log 2>&1
