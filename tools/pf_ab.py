"""A/B of the token-rich tiles on the prefill / 70B shapes: the non-persistent tcgen05 tile (BN 256,
the analytic choice) against the persistent tile at 128 and 192 tokens, timed like tools/tune.py
(graph of chained launches over 2 packed-weight copies, median of replays, per launch).

  python tools/pf_ab.py [--set prefill,70b] [--out gpurun_out/pf_ab.jsonl]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2508_19087_b200 as P  # noqa: E402
from tune import SETS, time_cfg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", default="prefill")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    P.clear_table()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    log = open(args.out, "a") if args.out else None
    for (m, n, k, wb, ab) in [c for nm in args.set.split(",") for c in SETS[nm]]:
        Ws = []
        for _ in range(2):
            c = torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), generator=g, device=dev, dtype=torch.int8)
            Ws.append(P.pack(c, wb, tiled=True))
        a = torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), generator=g, device=dev, dtype=torch.int8)
        A = P.pack(a, ab, digits=True)
        wsc = torch.exp2(torch.empty(n, device=dev).uniform_(-10, -6, generator=g))
        asc = torch.exp2(torch.empty(m, device=dev).uniform_(-6, -2, generator=g))
        out = torch.empty((m, n), dtype=torch.float16, device=dev)
        base = P.select_config(m, n, k, wb, ab)
        rec = {"M": m, "N": n, "K": k, "W": wb, "A": ab, "lib": os.environ.get("APT_LIB_VARIANT", "libapt.so")}
        cfgs = {"tc256": base}
        for bn in (128, 192, 256):
            cfgs[f"pf{bn}"] = dict(base, kernel=6, bm=128, bn=bn, bk=128, stages={128: 6, 192: 4, 256: 3}[bn], split_k=1,
                                   cta_pair=0, cluster_n=1, mma_kind=0)
        for name, cfg in cfgs.items():
            rec[name] = round(time_cfg(Ws, A, wsc, asc, out, cfg, st, 10), 2)
        ops = 2.0 * m * n * k
        rec["best_tops"] = round(ops / min(rec[x] for x in cfgs) * 1e-6, 1)
        print(json.dumps(rec), flush=True)
        if log:
            log.write(json.dumps(rec) + "\n")
        del Ws, A, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
