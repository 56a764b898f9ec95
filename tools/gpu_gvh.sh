set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
APT_LIB_VARIANT=libapt_gvh.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k gemv > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
for v in libapt.so libapt_gvh.so libapt.so libapt_gvh.so; do
APT_LIB_VARIANT=$v timeout 600 python tools/gemv_nw.py >> gpurun_out/gvnw_${T}_$v.log 2>&1
done
