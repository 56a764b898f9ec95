"""Activation pack timing on the token-rich shapes (digit view on): device time per launch, one launch
after a 256 MB L2 flush (the bench's prefill-leg method) and 10 chained launches without a flush.

  [APT_LIB_VARIANT=...] python tools/pack_ab.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2508_19087_b200 as P  # noqa: E402
from bench import _chain_us  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
nof = torch.empty(1, dtype=torch.uint8, device=dev)
for (m, k, ab) in ((2048, 4096, 8), (2048, 11008, 8), (2048, 4096, 4), (2048, 11008, 4), (4096, 8192, 4)):
    a = torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), device=dev, dtype=torch.int8)
    A = P.pack(a, ab, digits=True)
    cold = _chain_us(torch, st, lambda: P.pack(a, ab, out=A), 1, 7, flush)
    warm = _chain_us(torch, st, lambda: [P.pack(a, ab, out=A) for _ in range(10)], 10, 7, nof)
    byt = m * k + A.planes.numel() * 4 + A.digits.numel() + A.row_sum.numel() * 4
    print(json.dumps({"lib": os.environ.get("APT_LIB_VARIANT", "libapt.so"), "M": m, "K": k, "A": ab,
                      "cold_us": round(cold, 2), "warm_us": round(warm, 2), "MB": round(byt / 1e6, 1),
                      "cold_GBs": round(byt / cold / 1e3, 1)}), flush=True)
