# Final evidence session: parity, smoke, bench line, reference arm, decode kernel table, ncu launch list + traffic.
set +e
cd $GRAFT_REPO_ROOT
TAG=${1:-final}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1
rm -f gpurun_out/kernels_${TAG}_decode.jsonl
timeout 600 python tools/bench_kernels.py --suite decode --out gpurun_out/kernels_${TAG}_decode.jsonl > gpurun_out/kernels_${TAG}_decode.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-baselines > gpurun_out/bench_ncu_$TAG.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"gemm_tc|gemv|skinny" -s 72 -c 36 --csv --log-file gpurun_out/traffic_$TAG.csv python bench.py --steps 1 --warmup 3 --no-baselines > gpurun_out/bench_ncu2_$TAG.log 2>&1
