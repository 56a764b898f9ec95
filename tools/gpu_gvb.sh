set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
for v in libapt.so libapt_gvb.so libapt_gvc.so libapt.so libapt_gvb.so libapt_gvc.so; do
GV_MS=1 APT_LIB_VARIANT=$v timeout 600 python tools/gemv_ab.py >> gpurun_out/gv_${T}_$v.log 2>&1
done
