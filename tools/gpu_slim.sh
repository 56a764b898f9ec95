set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
APT_LIB_VARIANT=libapt_slim.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "decode or llama7b or config or f16 or random" > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
for v in libapt.so libapt_slim.so; do
APT_LIB_VARIANT=$v timeout 300 python tools/bench_kernels.py --suite decode --out gpurun_out/kern_${T}_$v.jsonl > /dev/null 2>&1
done
APT_LIB_VARIANT=libapt_slim.so timeout 600 python bench.py --no-baselines > gpurun_out/bench_${T}_slim.log 2>&1
timeout 600 python bench.py --no-baselines > gpurun_out/bench_${T}_base.log 2>&1
