set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python tools/bench_kernels.py --suite prefill --out gpurun_out/pre_$T.jsonl > /dev/null 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
