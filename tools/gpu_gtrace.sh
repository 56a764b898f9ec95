set +e
cd $GRAFT_REPO_ROOT
TAG=${1:-gt}
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
rm -f gpurun_out/gtrace_$TAG.log
for v in libapt_gtrace.so libapt_gtrace_late.so; do
for c in "16 4096 4096 2 2" "16 11008 4096 2 2" "1 4096 11008 4 4" "16 4096 4096 2 2 4" "16 4096 4096 2 2 2"; do
  echo "== $v $c" >> gpurun_out/gtrace_$TAG.log
  APT_LIB_VARIANT=$v timeout 120 python tools/tc_gtrace.py $c >> gpurun_out/gtrace_$TAG.log 2>&1
done
done
timeout 300 python tools/bench_kernels.py --suite decode > gpurun_out/kern_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1
