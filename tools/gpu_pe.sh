set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
for v in libapt.so libapt_oldph.so libapt.so libapt_oldph.so; do
APT_LIB_VARIANT=$v timeout 300 python tools/bench_kernels.py --suite prefill --out gpurun_out/pre_${T}_$v.jsonl > /dev/null 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
