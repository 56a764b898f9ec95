set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$TAG.log
for c in "1 11008 4096 1 2" "1 4096 2048 1 2 1"; do
  echo "== $c" >> gpurun_out/tr_$TAG.log
  APT_LIB_VARIANT=libapt_trace.so timeout 120 python tools/tc_trace.py $c 2>&1 | head -20 >> gpurun_out/tr_$TAG.log
done
for v in libapt.so libapt_n2.so libapt_n1.so; do
  APT_LIB_VARIANT=$v timeout 300 python tools/bench_kernels.py --suite decode --out gpurun_out/kern_${TAG}_$v.jsonl > gpurun_out/kern_${TAG}_$v.log 2>&1
done
