# Round-evidence session: parity, smoke, bench line, GEMV A/B, ncu launch list + traffic + full captures.
set +e
cd $GRAFT_REPO_ROOT
TAG=${1:-full}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:skinny -s 2 -c 1 -o gpurun_out/prof_sk_$TAG python tools/prof_one.py 8 11008 4096 4 4 4 > gpurun_out/ncu_sk_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-baselines > gpurun_out/bench_ncu_$TAG.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"gemm_tc|gemv|skinny" -s 72 -c 36 --csv --log-file gpurun_out/traffic_$TAG.csv python bench.py --steps 1 --warmup 3 --no-baselines > gpurun_out/bench_ncu2_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemv -s 2 -c 1 -o gpurun_out/prof_gemv_$TAG python tools/prof_one.py 1 11008 4096 4 4 4 > gpurun_out/ncu_gemv_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/prof_dec_$TAG python tools/prof_one.py 16 11008 4096 4 4 4 > gpurun_out/ncu_dec_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/prof_pre_$TAG python tools/prof_one.py 2048 4096 4096 4 4 4 > gpurun_out/ncu_pre_$TAG.log 2>&1
