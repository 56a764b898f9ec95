set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1
for v in libapt_trace.so libapt_tr_nomma.so; do
for c in "1 4096 2048 1 2 1" "1 4096 2048 4 4 1" "16 4096 2048 1 2 1"; do
  echo "== $v $c" >> gpurun_out/tr_$TAG.log
  APT_LIB_VARIANT=$v timeout 120 python tools/tc_trace.py $c 2>&1 | head -20 >> gpurun_out/tr_$TAG.log
done
done
