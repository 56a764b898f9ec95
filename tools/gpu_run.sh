# GPU session script (edited per call)
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"gemm|gemv" -s 72 -c 36 --csv --log-file gpurun_out/traffic_r2.csv python bench.py --steps 2 --warmup 3 --no-baselines --legs none > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-baselines --legs none > /dev/null 2>&1
timeout 300 ncu --set full --import-source on -k regex:gemm_dec -s 2 -c 1 -o gpurun_out/r2_ncu_dec_m16 -f python tools/prof_one.py 16 4096 4096 2 2 3 0 kernel=5,bm=32,stages=8,split_k=1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/r2_ncu_tcdec_m16 -f python tools/prof_one.py 16 11008 4096 4 4 3 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on -k regex:gemv -s 2 -c 1 -o gpurun_out/r2_ncu_gemv_m1 -f python tools/prof_one.py 1 11008 4096 4 4 3 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on -k regex:gemm_tc -s 1 -c 1 -o gpurun_out/r2_ncu_prefill -f python tools/prof_one.py 2048 4096 4096 4 4 3 > /dev/null 2>&1
ls gpurun_out
