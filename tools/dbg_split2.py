import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P
from oracle import apt_oracle as O
from synth import signed_codes

def stg(wb, bn):
    cw = 8 if wb <= 4 else 4
    slots = 6 if bn <= 64 else 2
    v = ((108 if bn <= 128 else 216) * 1024 - slots * wb * 128 * cw * 4 - (128 * (bn + 8) * 4 if bn <= 64 else 0) - 4096) // (bn * 128)
    return max(2, min(8, v))

m, n, k, pa, pw = 2, 8, 2048, 4, 4
a = signed_codes(m, k, pa, seed=1); w = signed_codes(n, k, pw, seed=2)
A = P.pack(torch.from_numpy(a).cuda(), pa, digits=True); W = P.pack(torch.from_numpy(w).cuda(), pw)
ref = O.gemm_signed(a, w)
ua = O.offset_bits_matrix(a, pa); uw = O.offset_bits_matrix(w, pw)
U = ua @ uw.T
half = k // 2
U0 = ua[:, :half] @ uw[:, :half].T; U1 = U - U0
for split in (1, 2):
    cfg = dict(P.select_config(m, n, k, pw, pa), bn=16, split_k=split, cluster_n=1, stages=stg(pw, 16))
    y = P.gemm(W, A, config=cfg).cpu().numpy().astype(np.int64)
    print("split", split)
    print(" ref   ", ref[0, :8])
    print(" got   ", y[0, :8])
    print(" ref-got", (ref - y)[0, :8])
    print(" U0    ", U0[0, :8], " U1", U1[0, :8], " U", U[0, :8])
