"""mma.sync skinny GEMM (APT_KERNEL_SKINNY, warps 4/8/16) vs the selector's kernel at M = 1..16."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_kernels import case  # noqa: E402
import paper_2508_19087_b200 as P  # noqa: E402

for m in [int(x) for x in os.environ.get("SK_MS", "8,16").split(",")]:
    for wb, ab in ((1, 2), (2, 2), (3, 4), (4, 4)):
        for n, k in ((4096, 4096), (11008, 4096), (4096, 11008)):
            base = P.select_config(m, n, k, wb, ab)
            r = {"M": m, "N": n, "K": k, "wb": wb, "ab": ab, "sel_kernel": base["kernel"],
                 "sel_us": case(m, n, k, wb, ab, cfg=base, baselines=False)["gemm_us"]}
            for warps in (4, 8, 16):
                cfg = dict(base, kernel=4, bm=16, bn=8 if m <= 8 else 16, bk=256, split_k=warps, stages=1,
                           cta_pair=0, cluster_n=1)
                r[f"sk{warps}_us"] = case(m, n, k, wb, ab, cfg=cfg, baselines=False)["gemm_us"]
            print(json.dumps(r), flush=True)
