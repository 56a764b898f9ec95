set -x
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/b_final10.json 2> gpurun_out/b_final10.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke10.txt 2>&1
B="python bench.py --steps 2 --warmup 1 --legs none --no-baselines"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_grp -c 1 --csv --log-file gpurun_out/traffic_grp10.csv $B > gpurun_out/ncu_t10.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_grp10.csv $B > gpurun_out/ncu_l10.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_grp -c 1 -o gpurun_out/grp_bench_all10 -f $B > gpurun_out/ncu_f10.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gputest_final10.txt
cat gpurun_out/gputest_final10.txt gpurun_out/smoke10.txt
