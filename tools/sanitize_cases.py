"""Small launches of every kernel family (pack, quantize-pack, GEMV, skinny, tcgen05 decode split-K and
prefill tiles, kind::mxf4, the register-fed decode GEMM with and without split-K tickets, the persistent
tile, expand passes, the ablation's recombine) for compute-sanitizer runs; checks each result against the
oracle.  Run with APT_TABLE=none so the analytic configs are the ones named here."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402
from oracle import apt_oracle as O  # noqa: E402
from synth import fp16_activations, signed_codes  # noqa: E402

dev = torch.device("cuda:0")


def run(m, n, k, wb, ab, digits=True, tiled=True, **over):
    a = signed_codes(m, k, ab, seed=m + k)
    w = signed_codes(n, k, wb, seed=n + k)
    A = P.pack(torch.from_numpy(a).to(dev), ab, digits=digits)
    W = P.pack(torch.from_numpy(w).to(dev), wb, tiled=tiled)
    cfg = P.select_config(m, n, k, wb, ab)
    if over:
        cfg = dict(cfg, **over)
    y = P.gemm(W, A, config=cfg).cpu().numpy().astype(np.int64)
    assert np.array_equal(y, O.gemm_signed(a, w)), (m, n, k, wb, ab, cfg)
    print("ok", m, n, k, wb, ab, "kernel", cfg["kernel"], "split", cfg["split_k"], "bn", cfg["bn"], flush=True)


run(1, 300, 700, 3, 4)            # GEMV
run(2, 4096, 512, 2, 2)           # GEMV, 16 warps
run(5, 333, 1000, 4, 4)           # skinny
run(16, 256, 4096, 2, 2)          # tcgen05 decode, split-K cluster
run(40, 256, 2048, 4, 4)          # tcgen05 BN 64
run(300, 384, 1024, 4, 8)         # tcgen05 prefill tile
run(16, 256, 1024, 2, 2, digits=False)  # expand pass into the workspace
run(16, 300, 2048, 2, 2, kernel=5, bm=32, bn=16, bk=256, stages=8, split_k=1, cluster_n=1)   # DEC
run(5, 300, 2048, 4, 4, kernel=5, bm=32, bn=8, bk=256, stages=4, split_k=3, cluster_n=1)     # DEC split-K tickets
run(300, 333, 1300, 3, 3, kernel=2, bn=256, stages=5, split_k=1, cluster_n=1, mma_kind=1)     # tcgen05 kind::mxf4
run(300, 333, 1300, 4, 4, kernel=6, bm=128, bn=128, bk=128, stages=6, split_k=1, cluster_n=1)  # persistent i8
run(300, 333, 1300, 2, 3, kernel=6, bm=128, bn=128, bk=128, stages=6, split_k=1, cluster_n=1, mma_kind=1)  # persistent mxf4
from paper_2508_19087_b200 import ablation  # noqa: E402
a = signed_codes(16, 500, 2, seed=3)
w = signed_codes(64, 500, 3, seed=4)
pp = ablation.PlanePairs(torch.from_numpy(a).to(dev), 2, torch.from_numpy(w).to(dev), 3)
assert np.array_equal(pp.basic().cpu().numpy().astype(np.int64), O.gemm_bipolar(a, 2, w, 3))
print("ok ablation recombine", flush=True)
x = fp16_activations(3, 1000, seed=1)
Pk, s = P.quantize_pack(torch.from_numpy(x).to(dev), 4)
codes, so = O.quantize_symmetric(x, 4)
assert np.array_equal(s.cpu().numpy(), so)
torch.cuda.synchronize()
print("sanitize cases ok")
