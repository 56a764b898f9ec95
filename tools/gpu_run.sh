# GPU session script (edited per call)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2_gputest2.txt
timeout 300 python tools/pack_bench.py > gpurun_out/r2_pack_bench2.jsonl 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --no-baselines > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err
cat gpurun_out/r2_gputest2.txt; head -14 gpurun_out/r2_pack_bench2.jsonl
