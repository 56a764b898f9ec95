set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
timeout 300 python tools/bench_kernels.py --suite prefill --out gpurun_out/pre_${T}_def.jsonl > /dev/null 2>&1
timeout 300 python tools/bench_kernels.py --suite prefill --bn 256 --cn 1 --out gpurun_out/pre_${T}_256c1.jsonl > /dev/null 2>&1
timeout 300 python tools/bench_kernels.py --suite prefill --bn 256 --cn 2 --out gpurun_out/pre_${T}_256c2.jsonl > gpurun_out/pre_${T}.log 2>&1
