set +e
cd $GRAFT_REPO_ROOT
TAG=${1:-gt}
for c in "16 4096 4096 2 2" "16 11008 4096 4 4" "16 4096 4096 2 2 4"; do
  echo "== $c" >> gpurun_out/gtrace_$TAG.log
  APT_LIB_VARIANT=libapt_gtrace.so timeout 120 python tools/tc_gtrace.py $c >> gpurun_out/gtrace_$TAG.log 2>&1
done
timeout 240 python -m pytest tests -m gpu -q --timeout 60 -x > gpurun_out/pytest_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python tools/bench_kernels.py --suite decode > gpurun_out/kern_${TAG}_base.log 2>&1
set +e
cd $GRAFT_REPO_ROOT

for c in ; do
  echo "== $c" >> gpurun_out/trace_$TAG.log
  APT_LIB_VARIANT=libapt_trace.so timeout 120 python tools/tc_trace.py $c >> gpurun_out/trace_$TAG.log 2>&1
done
