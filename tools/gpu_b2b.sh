# Back-to-back timelines (gtrace build) + prefill BN sweep.
#   gpurun --timeout 900 -- bash tools/gpu_b2b.sh TAG
set +e
TAG=${1:-b2b}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in "16 4096 4096 2 2 6" "16 11008 4096 4 4 6" "1 4096 4096 1 2 6" "bench"; do
  echo "== $c" >> gpurun_out/b2b_$TAG.log
  APT_LIB_VARIANT=libapt_gtrace.so timeout 120 python tools/tc_gtrace_b2b.py $c >> gpurun_out/b2b_$TAG.log 2>&1
done
timeout 300 python tools/bench_kernels.py --suite prefill --bn 256 --cn 1 --out gpurun_out/kernels_${TAG}_pre256.jsonl > gpurun_out/kern_${TAG}_pre256.log 2>&1
timeout 300 python tools/bench_kernels.py --suite prefill --bn 256 --cn 2 --out gpurun_out/kernels_${TAG}_pre256c2.jsonl > gpurun_out/kern_${TAG}_pre256c2.log 2>&1
