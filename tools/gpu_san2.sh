set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_synccheck_$T.log 2>&1
echo "rc=$?" >> gpurun_out/san_synccheck_$T.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_racecheck_$T.log 2>&1
echo "rc=$?" >> gpurun_out/san_racecheck_$T.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_memcheck_$T.log 2>&1
echo "rc=$?" >> gpurun_out/san_memcheck_$T.log
timeout 300 python tools/bench_kernels.py --suite prefill --out gpurun_out/pre_$T.jsonl > /dev/null 2>&1
