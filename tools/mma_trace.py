"""CTA phase timeline of the decode kernel (needs libapt_mtrace.so built with -DAPT_MMA_TRACE),
plus the launch floor of back-to-back graph replays.

  python tools/mma_trace.py M,N,K,wb,ab ...
"""
import ctypes
import os
import sys

os.environ.setdefault("APT_LIB_VARIANT", "libapt_mtrace.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402

PH = "0 start | 1 first loads issued | 2 K loop done | 3 reduction barrier | 4 end"


def floor_us(fn, reps=200):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


dev = torch.device("cuda")
x = torch.zeros(1, device=dev)
print("graph floor, tiny torch kernel (x.add_(1)) us/launch:", round(floor_us(lambda: x.add_(1)), 3))
for spec in sys.argv[1:]:
    m, n, k, wb, ab = (int(v) for v in spec.split(","))
    Ws = [P.pack(torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), dtype=torch.int8, device=dev), wb)
          for _ in range(8)]
    A = P.pack(torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), dtype=torch.int8, device=dev), ab, digits=True)
    ws = torch.rand(n, device=dev)
    cfg = P.select_config(m, n, k, wb, ab)
    out = torch.empty((m, n), dtype=torch.float16, device=dev)
    for i in range(8):
        P.gemm(Ws[i], A, out_kind="f16", w_scale=ws, out=out)
    torch.cuda.synchronize()
    buf = np.zeros(4096 * 8, dtype=np.uint64)
    P._lib.lib().apt_debug_mma_trace(ctypes.c_void_p(buf.ctypes.data), 4096 * 8)
    ncta = min(4096, -(-n // cfg["bm"]) * -(-m // cfg["bn"]))
    t = buf.reshape(4096, 8)[:ncta, :5].astype(np.int64)
    rel = t - t[:, 0].min()
    print(f"== {spec} cfg={cfg} ctas={ncta}   phases: {PH}")
    for ph in range(5):
        col = rel[:, ph]
        print(f"  phase {ph}: min {col.min():7d} med {int(np.median(col)):7d} max {col.max():7d} ns")
    d = rel[:, 4] - rel[:, 0]
    print("  cta duration ns: min", d.min(), "med", int(np.median(d)), "max", d.max())
    print("  start quantiles ns:", [int(np.quantile(rel[:, 0], q)) for q in (0, .25, .5, .75, .9, 1.0)])
    j = [0]

    def run():
        P.gemm(Ws[j[0] % 8], A, out_kind="f16", w_scale=ws, out=out, config=cfg)
        j[0] += 1
    print("  graph back-to-back us/launch:", round(floor_us(run), 3))
