set +e
cd $GRAFT_REPO_ROOT
timeout 300 python tools/mma_trace.py 1,4096,4096,2,2 16,4096,4096,2,2 16,11008,4096,4,4 16,4096,11008,4,4 > gpurun_out/mtrace8.log 2>&1
timeout 600 python tools/time_cases.py 1,4096,4096,2,2 16,4096,4096,2,2 16,11008,4096,4,4 16,4096,11008,4,4 1,11008,4096,1,2 > gpurun_out/dec8.log 2>&1
echo done >> gpurun_out/dec8.log
