"""tcgen05 decode tile vs the mma.sync decode kernel (APT_KERNEL_MMA_SPLITK) at M = 8, 16."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_kernels import case  # noqa: E402
import paper_2508_19087_b200 as P  # noqa: E402

for m in (8, 16):
    for wb, ab in ((1, 2), (2, 2), (3, 4), (4, 4)):
        for n, k in ((4096, 4096), (11008, 4096), (4096, 11008)):
            tc = P.select_config(m, n, k, wb, ab)
            mm = dict(tc, kernel=1, bm=32, bk=256, bn=m if m <= 16 else 16, split_k=4, stages=2, cluster_n=1)
            r = {"M": m, "N": n, "K": k, "wb": wb, "ab": ab, "tc_us": case(m, n, k, wb, ab, cfg=tc, baselines=False)["gemm_us"]}
            try:
                r["mma_us"] = case(m, n, k, wb, ab, cfg=mm, baselines=False)["gemm_us"]
            except P._lib.AptError as e:
                r["mma_us"] = str(e)
            print(json.dumps(r), flush=True)
