set +e
cd $GRAFT_REPO_ROOT
TAG=${1:-tr}
for c in "16 11008 4096 4 4 3" "16 4096 4096 2 2 8"; do
  echo "== $c" >> gpurun_out/trace_$TAG.log
  APT_LIB_VARIANT=libapt_trace.so timeout 120 python tools/tc_trace.py $c >> gpurun_out/trace_$TAG.log 2>&1
done
