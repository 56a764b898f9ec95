import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P
from oracle import apt_oracle as O
from synth import signed_codes

def stg(wb, bn):
    cw = 8
    slots = (6 if wb <= 4 else 3) if bn <= 64 else 2
    v = ((108 if bn <= 128 else 216) * 1024 - slots * wb * 128 * cw * 4 - (128 * (bn + 8) * 4 if bn <= 64 else 0) - 4096) // (bn * 128)
    return max(2, min(8, v))

for (m, n, k, pa, pw) in [(24, 43, 261, 1, 2), (16, 200, 4096, 2, 2), (16, 4096, 4096, 2, 2), (1, 300, 2048, 4, 4)]:
    a = signed_codes(m, k, pa, seed=1); w = signed_codes(n, k, pw, seed=2)
    A = P.pack(torch.from_numpy(a).cuda(), pa, digits=True); W = P.pack(torch.from_numpy(w).cuda(), pw)
    ref = O.gemm_signed(a, w)
    for bn in (16, 64):
        for split in (1, 2, 3, 4, 8):
            cfg = dict(P.select_config(m, n, k, pw, pa), bn=bn, split_k=split, cluster_n=1, stages=stg(pw, bn))
            if bn < m: continue
            try:
                y = P.gemm(W, A, config=cfg).cpu().numpy().astype(np.int64)
                bad = (y != ref)
                print(m, n, k, pa, pw, "bn", bn, "split", split, "ok" if not bad.any() else f"BAD {bad.sum()} / {bad.size}; rows bad {np.unique(np.nonzero(bad)[1] // 128)} cols {np.unique(np.nonzero(bad)[0])[:20]}", flush=True)
            except Exception as e:
                print(m, n, k, "bn", bn, "split", split, "ERR", e)
