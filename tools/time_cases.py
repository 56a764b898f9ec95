"""Time a few GEMM cases (no baselines): python tools/time_cases.py "M,N,K,wb,ab[,bn]" ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_kernels import case  # noqa: E402
import paper_2508_19087_b200 as P  # noqa: E402

for spec in sys.argv[1:]:
    v = [int(x) for x in spec.split(",")]
    m, n, k, wb, ab = v[:5]
    cfg = None
    if len(v) > 5:
        cfg = P.select_config(m, n, k, wb, ab)
        if cfg["kernel"] == 2:
            bn = v[5]
            cfg["bn"] = bn
            stage = bn * 128 + wb * 128 * 16
            cfg["stages"] = max(2, min(6, ((110 if bn <= 128 else 220) * 1024) // stage))
        else:
            cfg["bn"], cfg["split_k"] = v[5], v[6]
    r = case(m, n, k, wb, ab, cfg=cfg, baselines=False, tag=os.environ.get("APT_LIB_VARIANT", "libapt.so"))
    print(json.dumps({k2: r[k2] for k2 in ("tag", "M", "N", "K", "wbits", "abits", "gemm_us", "eff_tops", "hbm_gbs", "config")}), flush=True)
