"""Decode GEMM time vs split_k for the tcgen05 kernel."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_kernels import case  # noqa
import paper_2508_19087_b200 as P  # noqa
for (m, n, k, wb, ab) in [(16, 4096, 4096, 2, 2), (16, 11008, 4096, 4, 4), (16, 4096, 11008, 4, 4), (1, 4096, 4096, 1, 2), (8, 11008, 4096, 2, 2), (16, 4096, 11008, 1, 2)]:
    for split in (1, 2, 3, 4, 5, 6, 8):
        cfg = dict(P.select_config(m, n, k, wb, ab), split_k=split)
        try:
            r = case(m, n, k, wb, ab, cfg=cfg, baselines=False)
        except P._lib.AptError:
            continue
        print(json.dumps({"M": m, "N": n, "K": k, "wb": wb, "ab": ab, "split": split, "gemm_us": r["gemm_us"], "GB/s": r["hbm_gbs"]}), flush=True)
