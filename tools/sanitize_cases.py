"""Small launches of every kernel family (pack, quantize-pack, GEMV, skinny, tcgen05 decode split-K and
prefill tiles, expand pass) for compute-sanitizer runs; checks each result against the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402
from oracle import apt_oracle as O  # noqa: E402
from synth import fp16_activations, signed_codes  # noqa: E402

dev = torch.device("cuda:0")


def run(m, n, k, wb, ab, digits=True, tiled=True):
    a = signed_codes(m, k, ab, seed=m + k)
    w = signed_codes(n, k, wb, seed=n + k)
    A = P.pack(torch.from_numpy(a).to(dev), ab, digits=digits)
    W = P.pack(torch.from_numpy(w).to(dev), wb, tiled=tiled)
    cfg = P.select_config(m, n, k, wb, ab)
    y = P.gemm(W, A).cpu().numpy().astype(np.int64)
    assert np.array_equal(y, O.gemm_signed(a, w)), (m, n, k, wb, ab, cfg)
    print("ok", m, n, k, wb, ab, "kernel", cfg["kernel"], "split", cfg["split_k"], "bn", cfg["bn"], flush=True)


run(1, 300, 700, 3, 4)            # GEMV
run(2, 4096, 512, 2, 2)           # GEMV, 16 warps
run(5, 333, 1000, 4, 4)           # skinny
run(16, 256, 4096, 2, 2)          # tcgen05 decode, split-K cluster
run(40, 256, 2048, 4, 4)          # tcgen05 BN 64
run(300, 384, 1024, 4, 8)         # tcgen05 prefill tile
run(16, 256, 1024, 2, 2, digits=False)  # expand pass into the workspace
x = fp16_activations(3, 1000, seed=1)
Pk, s = P.quantize_pack(torch.from_numpy(x).to(dev), 4)
codes, so = O.quantize_symmetric(x, 4)
assert np.array_equal(s.cpu().numpy(), so)
torch.cuda.synchronize()
print("sanitize cases ok")
