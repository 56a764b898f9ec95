"""One grouped decode launch over the 36 BASELINE configs[1] cases (or a subset), for ncu captures.
usage: python tools/grp_once.py [W1A2|W2A2|W3A4|W4A4|all] [reps]"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402

SHAPES = [(4096, 4096), (11008, 4096), (4096, 11008)]
PREC = {"W1A2": (1, 2), "W2A2": (2, 2), "W3A4": (3, 4), "W4A4": (4, 4)}
which = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
precs = list(PREC.values()) if which == "all" else [PREC[which]]
dev = torch.device("cuda:0")
probs = []
for (wb, ab) in precs:
    for (n, k) in SHAPES:
        for m in (1, 8, 16):
            w = torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), dtype=torch.int8, device=dev)
            a = torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), dtype=torch.int8, device=dev)
            probs.append(dict(W=P.pack(w, wb, tiled=True), A=P.pack(a, ab, digits=True), out_kind="f16",
                              w_scale=torch.rand(n, device=dev) + 0.5, a_scale=torch.rand(m, device=dev) + 0.5))
ws = P.grouped_workspace(dev)
for _ in range(reps):
    P.gemm_grouped(probs, workspace=ws)
torch.cuda.synchronize()
print("ok", len(probs))
