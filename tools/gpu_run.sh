# GPU session script (edited per call)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "pf_" 2>&1 | tail -3 > gpurun_out/r2_pf_test.txt
timeout 900 python tools/tune.py --set prefill,70b --out /tmp/t.apt --log gpurun_out/r2_tune_log7.jsonl > /dev/null 2>&1
cat gpurun_out/r2_pf_test.txt
