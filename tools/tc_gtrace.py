"""Grid-wide globaltimer timeline of one TC-kernel launch (needs libapt_gtrace.so built with
-DAPT_TC_GTRACE): per-phase percentiles over CTAs, relative to the first CTA's entry.

  APT_LIB_VARIANT=libapt_gtrace.so python tools/tc_gtrace.py M N K wbits abits [split] [bn]
"""
import ctypes
import os
import sys

os.environ.setdefault("APT_LIB_VARIANT", "libapt_gtrace.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402

m, n, k, wb, ab = (int(v) for v in sys.argv[1:6])
dev = torch.device("cuda")
Ws = [P.pack(torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), dtype=torch.int8, device=dev), wb, tiled=True)
      for _ in range(2)]
A = P.pack(torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), dtype=torch.int8, device=dev), ab, digits=True)
ws = torch.rand(n, device=dev)
cfg = P.select_config(m, n, k, wb, ab)
if len(sys.argv) > 6:
    cfg["split_k"] = int(sys.argv[6])
if len(sys.argv) > 7:
    cfg["bn"] = int(sys.argv[7])
    cfg = [c for c in P.enumerate_configs(m, n, k, wb, ab) if c["kernel"] == 2 and c["bn"] == cfg["bn"]
           and c["split_k"] == cfg["split_k"] and c["cluster_n"] == 1 and c["mma_kind"] == 0][0]
out = torch.empty((m, n), dtype=torch.float16, device=dev)
flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)  # 256 MB, flushed by READING it (clean L2)
print("cfg", cfg)
names = ["entry", "prefetch", "w4start", "alloc0", "alloc1", "setup", "firstW", "tokens", "acc_full", "push", "received", "exit"]
cols = [0, 8, 12, 10, 11, 1, 2, 3, 4, 5, 9, 6]
for rep in range(4):
    fsum = flush.sum()
    P._lib.lib().apt_debug_tc_gtrace_reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    P.gemm(Ws[rep % 2], A, out_kind="f16", w_scale=ws, out=out, config=cfg)
    e1.record()
    torch.cuda.synchronize()
    buf = np.zeros(8192 * 16, dtype=np.uint64)
    P._lib.lib().apt_debug_tc_gtrace(ctypes.c_void_p(buf.ctypes.data), 8192 * 16)
    ntiles = -(-n // 128) * -(-m // cfg["bn"]) * cfg["split_k"]
    t = buf.reshape(8192, 16)[:ntiles].astype(np.int64)
    t0 = t[:, 0].min()
    print(f"rep {rep}: event {e0.elapsed_time(e1)*1e3:.2f} us, ctas {ntiles}, span {t[:, 6].max() - t0} ns, "
          f"sms {len(set(t[:, 7].tolist()))}")
    for nm, i in zip(names, cols):
        v = t[:, i] - t0
        v = v[t[:, i] > 0]
        if len(v):
            q = np.percentile(v, [0, 10, 50, 90, 100]).astype(int)
            print(f"  {nm:10s} " + " ".join(f"{x:7d}" for x in q))
