"""Small grouped launches for compute-sanitizer runs: apt_pack_grouped (codes and fp16 quantize) and
apt_gemm_grouped (mixed widths incl. split row tiles, every width class, group-wise scales, fused zero
points), each result checked against the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402
from oracle import apt_oracle as O  # noqa: E402
from synth import fp16_activations, signed_codes  # noqa: E402

dev = torch.device("cuda:0")


def d(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


# grouped packs
cases = [(1, 700, 2), (16, 4096, 4), (5, 257, 8)]
prs = [dict(codes=d(signed_codes(r, k, b, seed=r + k)), bits=b, out=P.alloc_packed(r, k, b, dev, digits=True))
       for (r, k, b) in cases]
prs += [dict(x=d(fp16_activations(r, k, seed=r)), bits=max(b, 2), out=P.alloc_packed(r, k, max(b, 2), dev, digits=True),
             scale=torch.empty(r, dtype=torch.float32, device=dev)) for (r, k, b) in cases]
P.pack_grouped(prs)
for pr, (r, k, b) in zip(prs[:3], cases):
    planes, _ = O.pack_planes(signed_codes(r, k, b, seed=r + k), b)
    assert np.array_equal(pr["out"].planes.cpu().numpy().view(np.uint32), planes)
print("ok pack_grouped", flush=True)

# grouped GEMMs: every width class, M <= 8 and M > 8, split tiles (more CTAs than units)
for wmax in (2, 4, 8):
    gcases = [(16, 300, 1000, wmax, 4), (1, 129, 513, 1, 2), (8, 77, 2600, min(wmax, 3), 8), (9, 256, 4096, 2, 2)]
    probs, refs = [], []
    for i, (m, n, k, pw, pa) in enumerate(gcases):
        a, w = signed_codes(m, k, pa, seed=i + 1), signed_codes(n, k, pw, seed=i + 50)
        probs.append(dict(W=P.pack(d(w), pw, tiled=True), A=P.pack(d(a), pa, digits=True)))
        refs.append(O.gemm_signed(a, w))
    for out, ref in zip(P.gemm_grouped(probs), refs):
        assert np.array_equal(out.cpu().numpy().astype(np.int64), ref)
    print("ok gemm_grouped wmax", wmax, flush=True)

# group-wise scales and fused zero points
m, n, k = 16, 300, 1000
a, w = signed_codes(m, k, 4, seed=3), signed_codes(n, k, 4, seed=4)
G = O.kpad(k) // 128
wg = np.full((G, n), 2.0 ** -8, dtype=np.float32)
A, W = P.pack(d(a), 4, digits=True), P.pack(d(w), 4, tiled=True)
got = P.gemm(W, A, out_kind="f16", w_gscale=d(wg)).cpu().numpy().astype(np.float64)
ref = O.group_dequant_gemm_fp64(a, w, wg)
assert (np.abs(got - ref) <= 2.0 ** -10 * np.abs(ref) + 2.0 ** -14).all()
ws, wz = np.full(n, 2.0 ** -8, dtype=np.float32), np.full(n, 2.0 ** -9, dtype=np.float32)
got = P.gemm(W, A, out_kind="f16", w_scale=d(ws), w_zero=d(wz)).cpu().numpy().astype(np.float64)
ref = O.dequant_gemm_fp64(a, w, ws, None, wz, None)
assert (np.abs(got - ref) <= 2.0 ** -9 * (np.abs(ref) + 1)).all()
torch.cuda.synchronize()
print("sanitize grouped ok", flush=True)
