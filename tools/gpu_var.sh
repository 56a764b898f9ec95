# A/B of in-tree library variants on the decode kernel suite.
#   gpurun -- bash tools/gpu_var.sh TAG libapt.so libapt_x.so ...
set +e
TAG=$1; shift
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "$@"; do
  APT_LIB_VARIANT=$v timeout 300 python tools/bench_kernels.py --suite decode --out gpurun_out/kern_${TAG}_$v.jsonl > gpurun_out/kern_${TAG}_$v.log 2>&1
done
