set +e
cd $GRAFT_REPO_ROOT
TAG=${1:-pre}
timeout 300 python tools/bench_kernels.py --suite prefill --bn 256 --cn 1 > gpurun_out/kern_${TAG}_bn256cn1.log 2>&1
timeout 300 python tools/bench_kernels.py --suite prefill --bn 256 --cn 2 > gpurun_out/kern_${TAG}_bn256cn2.log 2>&1
timeout 300 python tools/bench_kernels.py --suite prefill --bn 256 --cn 4 > gpurun_out/kern_${TAG}_bn256cn4.log 2>&1
timeout 300 python tools/bench_kernels.py --suite prefill --bn 128 --cn 2 > gpurun_out/kern_${TAG}_bn128cn2.log 2>&1
