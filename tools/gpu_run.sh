# GPU session script (edited per call)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "pack or digit or quant or repack or smoke" 2>&1 | tail -3 > gpurun_out/r2_pack_test.txt
timeout 600 python tools/pack_bench.py > gpurun_out/r2_pack_bench2.jsonl 2>&1
timeout 900 python bench.py --steps 50 --warmup 5 --no-baselines --legs none > gpurun_out/r2_bench8.json 2> gpurun_out/r2_bench8.err
cat gpurun_out/r2_pack_test.txt
