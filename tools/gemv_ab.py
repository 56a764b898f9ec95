"""GEMV (APT_KERNEL_GEMV) vs the tcgen05 decode kernel on the Llama-2-7B decode linears, M = 1..4."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_kernels import case  # noqa: E402
import paper_2508_19087_b200 as P  # noqa: E402

for m in [int(x) for x in os.environ.get("GV_MS", "1,2,4").split(",")]:
    for wb, ab in ((1, 2), (2, 2), (3, 4), (4, 4)):
        for n, k in ((4096, 4096), (11008, 4096), (4096, 11008)):
            tc = P.select_config(max(m, 3), n, k, wb, ab)  # the tensor-core decode tile (bn 16)
            gv = P.select_config(m, n, k, wb, ab) if m <= 2 else dict(
                tc, kernel=3, bm=32, bn=m, bk=128, split_k=8, stages=1, cta_pair=0, cluster_n=1)
            r_tc = case(m, n, k, wb, ab, cfg=tc, baselines=False)
            r_gv = case(m, n, k, wb, ab, cfg=gv, baselines=False)
            print(json.dumps({"M": m, "N": n, "K": k, "wb": wb, "ab": ab, "tc_us": r_tc["gemm_us"],
                              "gemv_us": r_gv["gemm_us"], "gemv_GBs": r_gv["hbm_gbs"]}), flush=True)
