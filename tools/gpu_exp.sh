set +e
cd $GRAFT_REPO_ROOT
TAG=${1:-ex}
for v in libapt_trace.so libapt_trace_spin.so; do
  for c in "16 4096 4096 2 2 4" "16 4096 4096 2 2 8"; do
    echo "== $v $c" >> gpurun_out/trace_$TAG.log
    APT_LIB_VARIANT=$v timeout 120 python tools/tc_trace.py $c >> gpurun_out/trace_$TAG.log 2>&1
  done
done
for v in libapt_gtrace.so libapt_gtrace_spin.so; do
for c in "16 4096 4096 2 2" "16 11008 4096 2 2" "16 4096 4096 2 2 4"; do
  echo "== $v $c" >> gpurun_out/gtrace_$TAG.log
  APT_LIB_VARIANT=$v timeout 120 python tools/tc_gtrace.py $c >> gpurun_out/gtrace_$TAG.log 2>&1
done
done
timeout 300 python tools/bench_kernels.py --suite decode > gpurun_out/kern_$TAG.log 2>&1
APT_LIB_VARIANT=libapt_spin.so timeout 300 python tools/bench_kernels.py --suite decode > gpurun_out/kern_spin_$TAG.log 2>&1
