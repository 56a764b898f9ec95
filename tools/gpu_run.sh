# GPU session script (edited per call)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "dec" 2>&1 | tail -2 > gpurun_out/r2_dec_test.txt
timeout 1500 python tools/tune.py --set decode --log gpurun_out/r2_tune_log8.jsonl > gpurun_out/r2_tune8.jsonl 2>&1
cp paper_2508_19087_b200/tables/b200.apt gpurun_out/b200.apt
timeout 900 python bench.py --steps 50 --warmup 5 --no-baselines --legs none > gpurun_out/r2_bench7.json 2> gpurun_out/r2_bench7.err
cat gpurun_out/r2_dec_test.txt
