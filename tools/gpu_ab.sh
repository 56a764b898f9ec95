set +e
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
VARS=${VARS:-"nte nte_bb1 bb1"}
for v in $VARS; do
  APT_LIB_VARIANT=libapt_$v.so timeout 240 python -m pytest tests -m gpu -q --timeout 60 -x > gpurun_out/pytest_${TAG}_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/pytest_${TAG}_$v.log
done
for rep in 1 2; do
timeout 300 python tools/bench_kernels.py --suite decode > gpurun_out/kern_${TAG}_base$rep.log 2>&1
for v in $VARS; do
APT_LIB_VARIANT=libapt_$v.so timeout 300 python tools/bench_kernels.py --suite decode > gpurun_out/kern_${TAG}_$v$rep.log 2>&1
done
done
