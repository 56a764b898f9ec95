set +e
cd $GRAFT_REPO_ROOT
TAG=${1:-nd}
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/prof_dec_$TAG python tools/prof_one.py 16 4096 4096 2 2 4 > gpurun_out/ncu_dec_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/prof_dec11k_$TAG python tools/prof_one.py 16 11008 4096 4 4 4 > gpurun_out/ncu_dec11k_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-baselines > gpurun_out/bench_ncu_$TAG.log 2>&1
