# One GPU session: parity tests, decode/prefill kernel timings, the bench line.
#   gpurun --timeout 1500 -- bash tools/gpu_session.sh TAG
set +e
TAG=${1:-run}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python tools/bench_kernels.py --suite decode > gpurun_out/kern_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
