"""GEMV time for 8 and 16 warps per CTA on the Llama-2-7B decode linears (M = 1)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_kernels import case  # noqa: E402
import paper_2508_19087_b200 as P  # noqa: E402

for wb, ab in ((1, 2), (2, 2), (3, 4), (4, 4)):
    for n, k in ((4096, 4096), (11008, 4096), (4096, 11008)):
        r = {"wb": wb, "ab": ab, "N": n, "K": k}
        for w in (8, 16):
            cfg = dict(P.select_config(1, n, k, wb, ab), split_k=w)
            r[f"nw{w}"] = case(1, n, k, wb, ab, cfg=cfg, baselines=False)["gemm_us"]
        print(json.dumps(r), flush=True)
