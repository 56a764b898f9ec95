# GPU session script (edited per call)
set -x
mkdir -p gpurun_out
timeout 1500 python tools/tune.py --set prefill,70b,sweep --log gpurun_out/r2_tune_log4.jsonl > gpurun_out/r2_tune4.jsonl 2>&1
cp paper_2508_19087_b200/tables/b200.apt gpurun_out/b200.apt
tail -2 gpurun_out/r2_tune4.jsonl
