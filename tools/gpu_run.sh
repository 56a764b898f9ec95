# GPU session script (edited per call)
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "tp_gemm or mxf4_matches" 2>&1 | tail -3 > gpurun_out/r2_tp_test.txt
( time timeout 900 python bench.py --steps 50 --warmup 5 ) > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err
tail -5 gpurun_out/r2_bench3.err; cat gpurun_out/r2_tp_test.txt
