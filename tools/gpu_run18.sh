set +e
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/pytest_gpu18.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu18.log
timeout 300 python tools/split_sweep.py > gpurun_out/split18.log 2>&1
for s in 1 2 8; do timeout 120 python tools/tc_trace.py 16 4096 4096 2 2 $s > gpurun_out/trace18_s$s.log 2>&1; done
