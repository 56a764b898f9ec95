set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k gemv > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
for v in libapt.so libapt_gv16.so libapt_gv8b3.so libapt_gv4b4.so; do
GV_MS=1,2 APT_LIB_VARIANT=$v timeout 600 python tools/gemv_ab.py > gpurun_out/gemv_${T}_$v.log 2>&1
done
