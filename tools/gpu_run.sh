# round-2 GPU session script (edited per call): tests, bench, ncu of the pack kernels
set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_gputest2.txt
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:pack_kernel -c 60 --csv python bench.py --steps 2 --warmup 3 --no-baselines > gpurun_out/r2_ncu_pack.csv 2>/dev/null
cat gpurun_out/r2_gputest2.txt; tail -c 400 gpurun_out/r2_bench2.json
