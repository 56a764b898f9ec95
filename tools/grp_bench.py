"""Time the grouped decode GEMM on the 36 BASELINE configs[1] cases vs the per-call chain.

Every problem has its OWN packed weights (3 copies per linear: M = 1, 8, 16 never share a weight
buffer) and two such sets alternate between replays, so weights come from HBM (2 x 400 MB > L2).
Prints one JSON line per variant: us per step, effective TOPS, algorithmic GB/s and HBM fraction."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402
from synth import log_uniform_scales, signed_codes  # noqa: E402

SHAPES = [(4096, 4096), (11008, 4096), (4096, 11008)]
PREC = [(1, 2), (2, 2), (3, 4), (4, 4)]
MS = [1, 8, 16]
dev = torch.device("cuda:0")
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6535.7


def kp(k):
    return -(-k // 256) * 256


def alg(m, n, k, wb, ab):
    return n * kp(k) * wb // 8 + m * kp(k) * ab // 8 + 8 * (m + n) + 2 * m * n


cases = [(m, n, k, wb, ab) for (wb, ab) in PREC for (n, k) in SHAPES for m in MS]
acts = {}
for (m, n, k, wb, ab) in cases:
    if (m, k, ab) not in acts:
        acts[(m, k, ab)] = (P.pack(torch.from_numpy(signed_codes(m, k, ab, seed=m + k + ab)).to(dev), ab, digits=True),
                            torch.from_numpy(log_uniform_scales(m, -6, -2, seed=m)).to(dev))
sets = []
for s in range(2):
    probs = []
    for i, (m, n, k, wb, ab) in enumerate(cases):
        w = torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), dtype=torch.int8, device=dev)
        W = P.pack(w, wb, tiled=True)
        A, asc = acts[(m, k, ab)]
        probs.append(dict(W=W, A=A, out_kind="f16", w_scale=torch.rand(n, device=dev) * 1e-3 + 1e-4, a_scale=asc,
                          out=torch.empty((m, n), dtype=torch.float16, device=dev)))
    sets.append(probs)
    del w
torch.cuda.synchronize()
ws = P.grouped_workspace(dev)
ops = sum(2 * m * n * k for (m, n, k, wb, ab) in cases)
byt = sum(alg(*c) for c in cases)
stream = torch.cuda.Stream()


def time_variant(name, fn, reps=50):
    try:
        _time_variant(name, fn, reps)
    except Exception as exc:  # e.g. a group larger than an experiment build's capacity
        print(json.dumps({"variant": name, "error": repr(exc)[:200]}), flush=True)


def _time_variant(name, fn, reps=50):
    with torch.cuda.stream(stream):
        fn(0)
        fn(1)
        torch.cuda.synchronize()
        gs = []
        for s in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                fn(s)
            gs.append(g)
        for j in range(6):
            gs[j % 2].replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for j in range(reps):
            gs[j % 2].replay()
        e1.record(stream)
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(json.dumps({"variant": name, "us_per_step": round(us, 2), "eff_tops": round(ops / us / 1e6, 2),
                      "alg_GBs": round(byt / us / 1e3, 1), "hbm_frac": round(byt / us / 1e3 / peak, 4)}), flush=True)


def per_call(s):
    for pr in sets[s]:
        P.gemm(pr["W"], pr["A"], out_kind="f16", w_scale=pr["w_scale"], a_scale=pr["a_scale"], out=pr["out"])


def grouped_all(s):
    P.gemm_grouped(sets[s], workspace=ws, stream=stream)


def grouped_prec(s):
    for i in range(4):
        P.gemm_grouped(sets[s][9 * i:9 * i + 9], workspace=ws, stream=stream)


time_variant("per_call_chain", per_call)
time_variant("grouped_1_launch", grouped_all)
time_variant("grouped_per_precision_4_launches", grouped_prec)

if len(sys.argv) > 1 and sys.argv[1] == "subsets":
    def sub(idx, name):
        ops_s = sum(2 * m * n * k for i, (m, n, k, wb, ab) in enumerate(cases) if i in idx)
        byt_s = sum(alg(*c) for i, c in enumerate(cases) if i in idx)

        def fn(s):
            P.gemm_grouped([sets[s][i] for i in idx], workspace=ws, stream=stream)
        global ops, byt
        o, b = ops, byt
        ops, byt = ops_s, byt_s
        time_variant(name, fn)
        ops, byt = o, b
    for pi, (wb, ab) in enumerate(PREC):
        sub([i for i, c in enumerate(cases) if (c[3], c[4]) == (wb, ab)], f"grouped_W{wb}A{ab}")
    for m in MS:
        sub([i for i, c in enumerate(cases) if c[0] == m], f"grouped_M{m}")

if len(sys.argv) > 1 and sys.argv[1] == "single":
    def single_chain(s):
        for pr in sets[s]:
            P.gemm_grouped([pr], workspace=ws, stream=stream)
    time_variant("grouped_single_problem_chain_36_launches", single_chain)
    # per case: chained 36 launches of the same case (like tools/tune.py), grouped vs the selector's apt_gemm
    for i, c in enumerate(cases):
        pr0, pr1 = sets[0][i], sets[1][i]
        ops1 = 2 * c[0] * c[1] * c[2]

        def t_of(fn, n=40):
            with torch.cuda.stream(stream):
                for j in range(4):
                    fn(j)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(stream)
                for j in range(n):
                    fn(j)
                e1.record(stream)
                torch.cuda.synchronize()
            return e0.elapsed_time(e1) * 1e3 / n
        tg = t_of(lambda j: P.gemm_grouped([pr0 if j % 2 else pr1], workspace=ws, stream=stream))
        tc = t_of(lambda j: P.gemm((pr0 if j % 2 else pr1)["W"], pr0["A"], out_kind="f16", w_scale=pr0["w_scale"],
                                    a_scale=pr0["a_scale"], out=pr0["out"], stream=stream))
        print(json.dumps({"case": c, "grouped_us": round(tg, 2), "apt_gemm_us": round(tc, 2)}), flush=True)
