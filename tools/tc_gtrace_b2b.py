"""Back-to-back globaltimer timeline of a CUDA graph of TC-kernel launches (needs an in-tree build with
-DAPT_TC_GTRACE, selected with APT_LIB_VARIANT): for each launch, when its CTAs enter, pass
griddepcontrol.wait, see the tokens / the accumulator / the split-K partials, and exit, relative to
the first launch's first entry (ns, percentiles over CTAs).

  APT_LIB_VARIANT=libapt_gtrace.so python tools/tc_gtrace_b2b.py M N K wbits abits [launches]
  APT_LIB_VARIANT=libapt_gtrace.so python tools/tc_gtrace_b2b.py bench     # the bench's 36-GEMM phase
"""
import ctypes
import os
import sys

os.environ.setdefault("APT_LIB_VARIANT", "libapt_gtrace.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402

dev = torch.device("cuda")
L = P._lib.lib()


def codes(rows, k, b):
    return torch.randint(-(1 << (b - 1)), 1 << (b - 1), (rows, k), dtype=torch.int8, device=dev)


if sys.argv[1] == "bench":
    cases = [(m, wb, ab, n, k) for m in (1, 8, 16) for (wb, ab) in ((1, 2), (2, 2), (3, 4), (4, 4))
             for (n, k) in ((4096, 4096), (11008, 4096), (4096, 11008))]
else:
    m, n, k, wb, ab = (int(v) for v in sys.argv[1:6])
    cases = [(m, wb, ab, n, k)] * (int(sys.argv[6]) if len(sys.argv) > 6 else 6)
Wc = {}
launches = []
for i, (m, wb, ab, n, k) in enumerate(cases):
    key = (wb, n, k, i % 4)
    if key not in Wc:
        Wc[key] = P.pack(codes(n, k, wb), wb, tiled=True)
    A = P.pack(codes(m, k, ab), ab, digits=True)
    out = torch.empty((m, n), dtype=torch.float16, device=dev)
    ws = torch.rand(n, device=dev)
    launches.append((Wc[key], A, out, ws, P.select_config(m, n, k, wb, ab)))


def step():
    for W, A, out, ws, cfg in launches:
        P.gemm(W, A, out_kind="f16", w_scale=ws, out=out, config=cfg)


step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.graph(g, stream=s):
    step()
flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)
for rep in range(3):
    fsum = flush.sum()
    torch.cuda.synchronize()
    L.apt_debug_tc_gtrace_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
print(f"graph of {len(cases)} launches: {e0.elapsed_time(e1) * 1e3:.2f} us (cold L2)")
buf = np.zeros(8192 * 16, dtype=np.uint64)
L.apt_debug_tc_gtrace(ctypes.c_void_p(buf.ctypes.data), 8192 * 16)
t = buf.reshape(8192, 16).astype(np.int64)
t = t[t[:, 0] > 0]
t = t[np.argsort(t[:, 0], kind="stable")]
t0 = t[0, 0]
names = [("entry", 0), ("setup", 1), ("pdlwait", 15), ("firstW", 2), ("tokens", 3), ("acc", 4), ("recv", 9),
         ("exit", 6)]
row = 0
print("launch  case                         ctas " + " ".join(f"{nm:>14s}" for nm, _ in names) + "   (p10/p90 ns)")
for i, (m, wb, ab, n, k) in enumerate(cases):
    G = int(t[row, 14])
    blk = t[row:row + G]
    row += G
    cols = []
    for nm, c in names:
        v = blk[:, c]
        v = v[v > 0] - t0
        cols.append(f"{int(np.percentile(v, 10)):6d}/{int(np.percentile(v, 90)):7d}" if len(v) else " " * 14)
    print(f"{i:5d}  M{m:<3d} W{wb}A{ab} {n:5d}x{k:<5d} {G:8d} " + " ".join(cols))
