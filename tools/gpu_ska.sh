set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
for v in libapt.so libapt_ska2.so libapt_ska4.so libapt_ska4b2.so; do
SK_MS=8,16 APT_LIB_VARIANT=$v timeout 600 python tools/skinny_ab.py > gpurun_out/sk_${T}_$v.log 2>&1
done
