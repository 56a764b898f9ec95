# Parity + smoke + kernel tables (prefill / 70b / sweep / decode) + bench line.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
for s in prefill 70b sweep decode; do
  rm -f gpurun_out/kernels_${T}_$s.jsonl
  timeout 600 python tools/bench_kernels.py --suite $s --out gpurun_out/kernels_${T}_$s.jsonl > gpurun_out/kernels_${T}_$s.log 2>&1
done
timeout 600 python bench.py > gpurun_out/bench_$T.log 2>&1
