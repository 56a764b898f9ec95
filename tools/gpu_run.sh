set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grouped.py -x -q 2>&1 | tail -3 > gpurun_out/grp_test.txt
timeout 600 python tools/grp_bench.py 2>&1 | grep "per_precision\|1_launch" >> gpurun_out/grp_test.txt
cat gpurun_out/grp_test.txt
