set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k skinny > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
SK_MS=1,8,16 timeout 900 python tools/skinny_ab.py > gpurun_out/sk_$T.log 2>&1
