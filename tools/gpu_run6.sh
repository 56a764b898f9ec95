set +e
cd $GRAFT_REPO_ROOT
for v in libapt.so libapt_e1.so libapt_e2.so libapt_e3.so; do
  APT_LIB_VARIANT=$v timeout 300 python tools/time_cases.py 2048,4096,4096,4,4 2048,4096,4096,4,4,256 2048,4096,4096,2,8 >> gpurun_out/exp6.log 2>&1
done
echo done >> gpurun_out/exp6.log
