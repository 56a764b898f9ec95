# GPU session script (edited per call)
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "ablation" 2>&1 | tail -3 > gpurun_out/r2_abl_test.txt
timeout 600 python tools/ablation.py > gpurun_out/r2_ablation.jsonl 2>&1
cat gpurun_out/r2_abl_test.txt gpurun_out/r2_ablation.jsonl
