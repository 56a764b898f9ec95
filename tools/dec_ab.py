"""A/B of decode GEMM configurations on the bench's 36 Llama-2-7B cases (BASELINE configs[1]).

Each measurement is a CUDA graph of R back-to-back launches of one case, every launch on its own
packed-weight copy (R copies > L2, so weights stream from HBM as in the bench), programmatic dependent
launch between them; time per launch = graph time / R (median of replays).  One JSON line per
(case, config).  Candidates: the selector's config and APT_KERNEL_DEC with every (bm, split) below.

  python tools/dec_ab.py [--cases all|M16|...] [--r 8]
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402

PREC = [(1, 2), (2, 2), (3, 4), (4, 4)]
SHAPES = [(4096, 4096), (11008, 4096), (4096, 11008)]
HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6555.2


def alg_bytes(m, n, k, wb, ab):
    kp = P.kpad(k)
    return n * kp * wb // 8 + m * kp * ab // 8 + 8 * (m + n) + 2 * m * n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1,8,16")
    ap.add_argument("--r", type=int, default=8)
    ap.add_argument("--dec", default="4:1,8:1,4:2,8:2,4:4")  # warps:split
    ap.add_argument("--reps", type=int, default=15)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    decs = [tuple(int(x) for x in v.split(":")) for v in args.dec.split(",") if v]
    for (n, k) in SHAPES:
        for (wb, ab) in PREC:
            Ws = []
            for r in range(args.r):
                c = torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), generator=g, device=dev, dtype=torch.int8)
                Ws.append(P.pack(c, wb, tiled=True))
                del c
            wsc = torch.exp2(torch.empty(n, device=dev).uniform_(-10, -6, generator=g))
            for m in [int(v) for v in args.ms.split(",")]:
                a = torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), generator=g, device=dev, dtype=torch.int8)
                A = P.pack(a, ab, digits=True)
                asc = torch.exp2(torch.empty(m, device=dev).uniform_(-6, -2, generator=g))
                out = torch.empty((m, n), dtype=torch.float16, device=dev)
                base = P.select_config(m, n, k, wb, ab)
                cands = [("selector", base)]
                if m <= 16:
                    for nw, sp in decs:
                        cands.append((f"dec w{nw}s{sp}", dict(base, kernel=5, bm=32, bn=8 if m <= 8 else 16, bk=256,
                                                              stages=nw, split_k=sp, cta_pair=0, cluster_n=1)))
                for name, cfg in cands:
                    def fn(cfg=cfg):
                        for W in Ws:
                            P.gemm(W, A, out_kind="f16", w_scale=wsc, a_scale=asc, out=out, config=cfg)
                    try:
                        fn()
                        torch.cuda.synchronize()
                        gr = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(gr, stream=st):
                            fn()
                        for _ in range(3):
                            gr.replay()
                        ts = []
                        for _ in range(args.reps):
                            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            e0.record(st)
                            gr.replay()
                            e1.record(st)
                            ts.append((e0, e1))
                        torch.cuda.synchronize()
                        us = statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3 / len(Ws)
                        print(json.dumps({"M": m, "N": n, "K": k, "W": wb, "A": ab, "cfg": name, "kernel": cfg["kernel"],
                                          "us": round(us, 3), "tops": round(2 * m * n * k / us / 1e6, 2),
                                          "hbm_frac": round(alg_bytes(m, n, k, wb, ab) / us / 1e3 / HBM, 4)}),
                              flush=True)
                    except Exception as exc:  # noqa: BLE001
                        print(json.dumps({"M": m, "N": n, "K": k, "W": wb, "A": ab, "cfg": name, "error": repr(exc)[:200]}),
                              flush=True)
            del Ws


if __name__ == "__main__":
    main()
