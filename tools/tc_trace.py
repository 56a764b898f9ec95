"""Per-stage timeline of one TC-kernel CTA (needs libapt_trace.so built with -DAPT_TC_TRACE)."""
import ctypes
import os
import sys

os.environ.setdefault("APT_LIB_VARIANT", "libapt_trace.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402

m, n, k, wb, ab = (int(v) for v in (sys.argv[1:6] if len(sys.argv) > 5 else (2048, 4096, 4096, 4, 4)))
dev = torch.device("cuda")
W = P.pack(torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), dtype=torch.int8, device=dev), wb, tiled=True)
A = P.pack(torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), dtype=torch.int8, device=dev), ab, digits=True)
ws = torch.rand(n, device=dev)
cfg = P.select_config(m, n, k, wb, ab)
if len(sys.argv) > 6:
    cfg["split_k"] = int(sys.argv[6])
print("cfg", cfg)
for _ in range(3):
    P.gemm(W, A, out_kind="f16", w_scale=ws, config=cfg)
torch.cuda.synchronize()
buf = np.zeros(8 * 512, dtype=np.int64)
rc = P._lib.lib().apt_debug_tc_trace(ctypes.c_void_p(buf.ctypes.data), 8 * 512)
t = buf.reshape(8, 512)
t0 = t[6, 0]
nk = (-(-k // 256) * 256) // 128
print("rc", rc, "setup", t[6, 1] - t0, "acc_full", t[5, 0] - t0, "pushed", t[5, 3] - t0, "cluster_barrier", t[5, 4] - t0,
      "epi_end", t[5, 1] - t0, "prod_end", t[5, 2] - t0)
print("ks  prod_issue  mma_full  mma_afull  conv_full  conv_done  conv_rebuilt")
for ks in range(nk):
    print(ks, *[int(t[s, ks] - t0) for s in (0, 1, 2, 3, 4, 7)])
