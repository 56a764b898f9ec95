"""Run one APT GEMM configuration a few times (for ncu captures).

  python tools/prof_one.py M N K wbits abits [reps] [bn] [key=value,...]
The optional last argument overrides config fields, e.g. kernel=5,bm=32,split_k=2 (APT_KERNEL_DEC: bn, bk
and stages are filled in).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402


def main():
    m, n, k, wb, ab = (int(v) for v in sys.argv[1:6])
    reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
    bn = int(sys.argv[7]) if len(sys.argv) > 7 else 0
    dev = torch.device("cuda")
    W = P.pack(torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), dtype=torch.int8, device=dev), wb, tiled=True)
    a = torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), dtype=torch.int8, device=dev)
    A = P.pack(a, ab, digits=True)
    ws = torch.rand(n, device=dev)
    cfg = P.select_config(m, n, k, wb, ab)
    if bn and cfg["kernel"] == 2:
        cfg["bn"] = bn
        stage = bn * 128 + wb * 128 * 16
        cfg["stages"] = max(2, min(6, ((110 if bn <= 128 else 220) * 1024) // stage))
    if len(sys.argv) > 8:
        for kv in sys.argv[8].split(","):
            key, v = kv.split("=")
            cfg[key] = int(v)
        if cfg["kernel"] == 2:  # tcgen05: the stage count follows (wbits, bn)
            match = [c for c in P.enumerate_configs(m, n, k, wb, ab)
                     if all(c[x] == cfg[x] for x in ("kernel", "bn", "split_k", "cluster_n", "mma_kind"))]
            if match:
                cfg = match[0]
        if cfg["kernel"] == 5:
            cfg.update(bm=32, bn=8 if m <= 8 else 16, bk=256, cta_pair=0, cluster_n=1)
    out = torch.empty((m, n), dtype=torch.float16, device=dev)
    for _ in range(reps):
        P.pack(a, ab, out=A)
        P.gemm(W, A, out_kind="f16", w_scale=ws, out=out, config=cfg)
    torch.cuda.synchronize()
    print("cfg", cfg)


if __name__ == "__main__":
    main()
