set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1
for v in libapt_trace.so libapt_tr_nowait.so libapt_tr_nomma.so; do
for c in "1 11008 4096 1 2" "16 11008 4096 4 4"; do
  echo "== $v $c" >> gpurun_out/tr_$TAG.log
  APT_LIB_VARIANT=$v timeout 120 python tools/tc_trace.py $c 2>&1 | head -14 >> gpurun_out/tr_$TAG.log
done
done
for v in libapt.so libapt_nowait.so libapt_nomma.so; do
  APT_LIB_VARIANT=$v timeout 300 python tools/bench_kernels.py --suite decode --out gpurun_out/kern_${TAG}_$v.jsonl > gpurun_out/kern_${TAG}_$v.log 2>&1
done
