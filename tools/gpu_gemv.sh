set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k gemv > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
timeout 600 python tools/gemv_ab.py > gpurun_out/gemv_$T.log 2>&1
