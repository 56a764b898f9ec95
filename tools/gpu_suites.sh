# Kernel tables for BASELINE configs[2..4] (prefill, 70B, precision sweep) vs cuBLAS.
#   gpurun --timeout 1200 -- bash tools/gpu_suites.sh TAG
set +e
TAG=${1:-suites}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for s in prefill 70b sweep; do
  timeout 400 python tools/bench_kernels.py --suite $s --out gpurun_out/kernels_${TAG}_$s.jsonl > gpurun_out/kern_${TAG}_$s.log 2>&1
done
