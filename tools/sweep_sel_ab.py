"""Selected-config timing of a few 4096^3 sweep cases (chained launches, tools/tune.py timing)."""
import os, sys, json, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import paper_2508_19087_b200 as P
from tune import time_cfg
dev = torch.device('cuda:0'); st = torch.cuda.Stream(); torch.cuda.set_stream(st)
g = torch.Generator(device=dev); g.manual_seed(3)
m = n = k = 4096
for (wb, ab) in ((1, 1), (2, 2), (2, 3), (3, 3), (1, 4), (4, 4), (8, 8)):
    Ws = [P.pack(torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), generator=g, device=dev, dtype=torch.int8), wb, tiled=True) for _ in range(2)]
    A = P.pack(torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), generator=g, device=dev, dtype=torch.int8), ab, digits=True)
    wsc = torch.ones(n, device=dev); asc = torch.ones(m, device=dev)
    out = torch.empty((m, n), dtype=torch.float16, device=dev)
    base = P.select_config(m, n, k, wb, ab)
    r = {"lib": os.environ.get("APT_LIB_VARIANT", "libapt.so"), "W": wb, "A": ab, "sel": base["kernel"], "sel_bn": base["bn"], "sel_mx": base["mma_kind"],
         "sel_us": round(time_cfg(Ws, A, wsc, asc, out, base, st, 10), 2)}
    print(json.dumps(r), flush=True)
