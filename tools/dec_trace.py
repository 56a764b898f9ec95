"""Per-warp globaltimer timeline of one APT_KERNEL_DEC launch (needs libapt_dtrace.so, built with
-DAPT_DEC_TRACE: python -c "from paper_2508_19087_b200 import _build; _build.build(out='.../libapt_dtrace.so',
defines=['APT_DEC_TRACE'])").  Prints, per phase, the min / median / max time (us) after the first warp's entry.

  python tools/dec_trace.py M N K wbits abits split warps [cold]
"""
import ctypes
import os
import sys

os.environ.setdefault("APT_LIB_VARIANT", "libapt_dtrace.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402

m, n, k, wb, ab, sp, nw = (int(v) for v in sys.argv[1:8])
cold = len(sys.argv) > 8 and sys.argv[8] == "cold"
dev = torch.device("cuda")
W = P.pack(torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), dtype=torch.int8, device=dev), wb, tiled=True)
A = P.pack(torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), dtype=torch.int8, device=dev), ab, digits=True)
ws = torch.rand(n, device=dev)
cfg = dict(P.select_config(m, n, k, wb, ab), kernel=5, bm=32, bn=8 if m <= 8 else 16, bk=256,
           stages=nw, split_k=sp, cta_pair=0, cluster_n=1)
L = P._lib.lib()
for _ in range(3):
    P.gemm(W, A, out_kind="f16", w_scale=ws, config=cfg)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
torch.cuda.synchronize()
L.apt_debug_dec_trace(None, 0, 1)
if cold:
    flush.fill_(1)
P.gemm(W, A, out_kind="f16", w_scale=ws, config=cfg)
torch.cuda.synchronize()
buf = np.zeros(8192 * 12, dtype=np.uint64)
L.apt_debug_dec_trace(ctypes.c_void_p(buf.ctypes.data), 8192 * 12, 0)
t = buf.reshape(8192, 12).astype(np.int64)
rows = int(t[0, 9])
t = t[:rows]
t0 = t[:, 0].min()
names = ["entry", "prologue", "pdl_wait", "first_tok", "first_w", "loop_done", "ticket", "exit", None, None, "summed", "kreduced"]
t = t[t[:, 0] > 0]
print("cfg", {k2: cfg[k2] for k2 in ("split_k", "stages")}, "warps", len(t), "SMs", len(set(t[:, 8])))
for i, nm in enumerate(names):
    if nm is None:
        continue
    v = t[:, i]
    v = v[v > 0] - t0
    if len(v):
        print(f"{nm:10s} min {v.min() / 1e3:7.2f}  med {np.median(v) / 1e3:7.2f}  max {v.max() / 1e3:7.2f} us")
