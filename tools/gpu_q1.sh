set +e
TAG=${1:-q1}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k quantize --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 120 ./tools/probe/launch_probe > gpurun_out/probe_$TAG.log 2>&1
