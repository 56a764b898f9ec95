set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
for v in libapt_trace.so libapt_trtok.so; do
for c in "1 11008 4096 1 2" "16 4096 4096 2 2"; do
  echo "== $v $c" >> gpurun_out/tr_$T.log
  APT_LIB_VARIANT=$v timeout 120 python tools/tc_trace.py $c 2>&1 | head -10 >> gpurun_out/tr_$T.log
done
done
for v in libapt.so libapt_tok.so; do
  APT_LIB_VARIANT=$v timeout 300 python tools/bench_kernels.py --suite decode --out gpurun_out/kern_${T}_$v.jsonl > gpurun_out/kern_${T}_$v.log 2>&1
done
timeout 600 python bench.py > gpurun_out/bench_$T.log 2>&1
APT_LIB_VARIANT=libapt_tok.so timeout 600 python bench.py --no-baselines > gpurun_out/bench_${T}_tok.log 2>&1
