set +e
cd $GRAFT_REPO_ROOT
timeout 300 python tools/mma_trace.py 1,16,4096,2,2 1,4096,4096,2,2 16,4096,4096,2,2 16,11008,4096,4,4 > gpurun_out/mtrace10.log 2>&1
