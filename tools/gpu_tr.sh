set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in "1 11008 4096 1 2" "1 11008 4096 4 4" "1 4096 4096 1 2" "16 11008 4096 4 4"; do
  echo "== $c" >> gpurun_out/tr_$1.log
  APT_LIB_VARIANT=libapt_trace.so timeout 120 python tools/tc_trace.py $c >> gpurun_out/tr_$1.log 2>&1
done
