# GPU session script (edited per call)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "mxf4" 2>&1 | tail -15 > gpurun_out/r2_mx_test.txt
cat gpurun_out/r2_mx_test.txt
timeout 1200 python tools/tune.py --set sweep --log gpurun_out/r2_tune_log3.jsonl > gpurun_out/r2_tune3.jsonl 2>&1
cp paper_2508_19087_b200/tables/b200.apt gpurun_out/b200.apt
timeout 300 ncu --set full --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/r2_mx_ncu -f python tools/prof_one.py 4096 4096 4096 3 3 3 0 kernel=2,bn=256,split_k=1,cluster_n=1,mma_kind=1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/r2_i8_ncu -f python tools/prof_one.py 4096 4096 4096 3 3 3 0 kernel=2,bn=128,split_k=1,cluster_n=1,mma_kind=0 > /dev/null 2>&1
