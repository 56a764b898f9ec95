set +e
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/pytest_gpu4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench4.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench4.log
timeout 900 python tools/bench_kernels.py --suite prefill --out gpurun_out/kernels4.jsonl > gpurun_out/kernels4.log 2>&1
echo "kern rc=$?" >> gpurun_out/kernels4.log
