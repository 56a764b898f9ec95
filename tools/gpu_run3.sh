set +e
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench3.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench3.log
