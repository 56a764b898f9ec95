"""Best Kernel Search (§5.2): time every legal configuration
(apt_enumerate_configs) of each problem key and write the fastest to an autotuned table that
apt_select_config consults (apt_table_load; format in include/apt.h).

Timing: a CUDA graph of R back-to-back apt_gemm launches (fp16 output with per-channel and per-token
scales, the bench's call), each on its own packed-weight copy so weights stream from HBM (R copies >
L2 for the decode shapes), programmatic dependent launch between them; median of replays, per launch.

  python tools/tune.py [--set decode|prefill|sweep|70b|all] [--out paper_2508_19087_b200/tables/b200.apt]
"""
import argparse
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2508_19087_b200 as P  # noqa: E402

LLAMA7B = [(4096, 4096), (11008, 4096), (4096, 11008)]
SETS = {
    "decode": [(m, n, k, wb, ab) for m in (1, 8, 16) for (wb, ab) in ((1, 2), (2, 2), (3, 4), (4, 4)) for (n, k) in LLAMA7B],
    "prefill": [(2048, n, k, wb, ab) for (wb, ab) in ((2, 8), (4, 4)) for (n, k) in LLAMA7B],
    "70b": [(4096, n, k, 2, 4) for (n, k) in ((8192, 8192), (28672, 8192))],
    "sweep": [(4096, 4096, 4096, wb, ab) for wb in range(1, 9) for ab in range(1, 9)],
}
KEYS = ("kernel", "w_digit", "a_digit", "bm", "bn", "bk", "stages", "split_k", "cta_pair", "cluster_n", "mma_kind")


def time_cfg(Ws, A, wsc, asc, out, cfg, st, reps):
    def fn():
        for W in Ws:
            P.gemm(W, A, out_kind="f16", w_scale=wsc, a_scale=asc, out=out, config=cfg)
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        fn()
    for _ in range(2):
        gr.replay()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        gr.replay()
        e1.record(st)
        ts.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ts) * 1e3 / len(Ws)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", default="decode")
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2508_19087_b200", "tables", "b200.apt"))
    ap.add_argument("--log", default=None)
    args = ap.parse_args()
    P.clear_table()  # time the explicit configs; the analytic choice is the baseline
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    names = list(SETS) if args.set == "all" else args.set.split(",")
    cases = [c for nm in names for c in SETS[nm]]
    rows, log = [], open(args.log, "a") if args.log else None
    wcache = {}
    t_start = time.time()
    for (m, n, k, wb, ab) in cases:
        big = m >= 1024
        ncopy = 2 if big else 8
        key = (n, k, wb, ncopy)
        if key not in wcache:
            wcache.clear()
            torch.cuda.empty_cache()
            Ws = []
            for _ in range(ncopy):
                c = torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), generator=g, device=dev, dtype=torch.int8)
                Ws.append(P.pack(c, wb, tiled=True))
                del c
            wcache[key] = Ws
        Ws = wcache[key]
        a = torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), generator=g, device=dev, dtype=torch.int8)
        A = P.pack(a, ab, digits=True)
        wsc = torch.exp2(torch.empty(n, device=dev).uniform_(-10, -6, generator=g))
        asc = torch.exp2(torch.empty(m, device=dev).uniform_(-6, -2, generator=g))
        out = torch.empty((m, n), dtype=torch.float16, device=dev)
        analytic = P.select_config(m, n, k, wb, ab)
        reps = 5 if big else 10
        best, best_us, res = None, float("inf"), []
        for cfg in P.enumerate_configs(m, n, k, wb, ab):
            try:
                us = time_cfg(Ws, A, wsc, asc, out, cfg, st, reps)
            except Exception as exc:  # noqa: BLE001
                res.append({"cfg": cfg, "error": repr(exc)[:120]})
                continue
            res.append({"cfg": cfg, "us": round(us, 3)})
            if us < best_us:
                best, best_us = cfg, us
        an_us = next((r["us"] for r in res if r.get("cfg") == analytic and "us" in r), None)
        rows.append((m, n, k, wb, ab, best, best_us, an_us))
        rec = {"M": m, "N": n, "K": k, "W": wb, "A": ab, "best": best, "best_us": round(best_us, 3),
               "analytic_us": an_us, "configs": len(res)}
        print(json.dumps(rec), flush=True)
        if log:
            log.write(json.dumps(dict(rec, all=res)) + "\n")
            log.flush()
        del A, a
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    old = []
    if os.path.exists(args.out):  # keep rows of keys not re-tuned now
        tuned = {r[:5] for r in rows}
        for line in open(args.out):
            f = line.split("#")[0].split()
            if len(f) != 17 or tuple(int(v) for v in f[:5]) in tuned:
                continue
            old.append(line.rstrip("\n"))
    with open(args.out, "w") as f:
        f.write("# apt-table v1 (include/apt.h apt_table_load): M N K wbits abits kernel w_digit a_digit bm bn bk "
                "stages split_k cta_pair cluster_n mma_kind us\n")
        f.write(f"# written by tools/tune.py on {torch.cuda.get_device_name(0)}; chained fp16-epilogue launches, "
                f"median per launch\n")
        for line in old:
            f.write(line + "\n")
        for (m, n, k, wb, ab, best, us, an) in rows:
            f.write(" ".join(str(v) for v in (m, n, k, wb, ab, *(best[x] for x in KEYS))) + f" {us:.3f}"
                    + (f"  # analytic {an:.3f}" if an else "") + "\n")
    print(json.dumps({"wrote": args.out, "rows": len(rows) + len(old), "seconds": round(time.time() - t_start, 1)}))


if __name__ == "__main__":
    main()
