set +e
cd $GRAFT_REPO_ROOT
timeout 600 python tools/bench_kernels.py --suite decode --out gpurun_out/kernels5_decode.jsonl > gpurun_out/kernels5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv python bench.py --steps 2 --warmup 1 --no-baselines > gpurun_out/ncu_launch5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_mma -s 2 -c 1 -o gpurun_out/prof_decode python tools/prof_one.py 16 4096 4096 2 2 3 > gpurun_out/ncu_dec.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/prof_tc python tools/prof_one.py 2048 4096 4096 4 4 3 > gpurun_out/ncu_tc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 4 -c 1 -o gpurun_out/prof_pack python tools/prof_one.py 2048 4096 4096 4 4 3 > gpurun_out/ncu_pack.log 2>&1
echo done
