"""One token-rich GEMM launch per config (for ncu): python tools/pf_once.py M N K W A [cfg...]
cfg in {tc256, pf128, pf192}; each is launched twice (warm-up + the captured one)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2508_19087_b200 as P  # noqa: E402

m, n, k, wb, ab = (int(x) for x in sys.argv[1:6])
names = sys.argv[6:] or ["tc256", "pf192"]
P.clear_table()
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(3)
c = torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), generator=g, device=dev, dtype=torch.int8)
W = P.pack(c, wb, tiled=True)
a = torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), generator=g, device=dev, dtype=torch.int8)
A = P.pack(a, ab, digits=True)
wsc = torch.exp2(torch.empty(n, device=dev).uniform_(-10, -6, generator=g))
asc = torch.exp2(torch.empty(m, device=dev).uniform_(-6, -2, generator=g))
out = torch.empty((m, n), dtype=torch.float16, device=dev)
base = P.select_config(m, n, k, wb, ab)
for name in names:
    cfg = dict(base) if name == "tc256" else dict(base, kernel=6, bm=128, bn=int(name[2:]), bk=128,
                                                      stages={"pf128": 6, "pf192": 4, "pf256": 3}[name], split_k=1, cta_pair=0,
                                                      cluster_n=1, mma_kind=0)
    for _ in range(2):
        P.gemm(W, A, out_kind="f16", w_scale=wsc, a_scale=asc, out=out, config=cfg)
    torch.cuda.synchronize()
print("ok")
