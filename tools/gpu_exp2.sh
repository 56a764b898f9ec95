set +e
cd $GRAFT_REPO_ROOT
TAG=${1:-ex}
VARS=${VARS:-"tf cp tfcp"}
for v in $VARS; do
  APT_LIB_VARIANT=libapt_$v.so timeout 240 python -m pytest tests -m gpu -q --timeout 60 -x > gpurun_out/pytest_${TAG}_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/pytest_${TAG}_$v.log
done
for v in gtrace $(for x in $VARS; do echo gtrace_$x; done); do
for c in "16 4096 4096 2 2" "16 11008 4096 4 4" "16 4096 4096 2 2 4"; do
  echo "== $v $c" >> gpurun_out/gtrace_$TAG.log
  APT_LIB_VARIANT=libapt_$v.so timeout 120 python tools/tc_gtrace.py $c >> gpurun_out/gtrace_$TAG.log 2>&1
done
done
timeout 300 python tools/bench_kernels.py --suite decode > gpurun_out/kern_${TAG}_base.log 2>&1
for v in $VARS; do
APT_LIB_VARIANT=libapt_$v.so timeout 300 python tools/bench_kernels.py --suite decode > gpurun_out/kern_${TAG}_$v.log 2>&1
done
