set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$T.log 2>&1
