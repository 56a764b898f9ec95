set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi_$T.log
for v in libapt.so libapt_nozpf.so libapt_oldph.so libapt.so libapt_nozpf.so libapt_oldph.so; do
APT_LIB_VARIANT=$v timeout 300 python tools/bench_kernels.py --suite prefill --out gpurun_out/pre_${T}_$v.jsonl > /dev/null 2>&1
done
