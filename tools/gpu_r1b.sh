# Re-entry session: parity, smoke, bench line, back-to-back decode timeline of the bench's GEMM phase.
#   gpurun --timeout 1500 -- bash tools/gpu_r1b.sh TAG
set +e
TAG=${1:-r1b}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
APT_LIB_VARIANT=libapt_gtrace.so timeout 120 python tools/tc_gtrace_b2b.py bench > gpurun_out/b2b_$TAG.log 2>&1
APT_LIB_VARIANT=libapt_gtrace.so timeout 120 python tools/tc_gtrace_b2b.py 16 4096 4096 2 2 6 >> gpurun_out/b2b_$TAG.log 2>&1
APT_LIB_VARIANT=libapt_gtrace.so timeout 120 python tools/tc_gtrace_b2b.py 16 11008 4096 4 4 6 >> gpurun_out/b2b_$TAG.log 2>&1
