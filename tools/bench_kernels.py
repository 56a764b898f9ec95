"""Per-configuration kernel timing (one JSON object per line) for BASELINE.json configs[1..4]:
APT GEMM time (CUDA graph of R launches, weights rotated over enough copies to exceed L2),
activation-pack time, and cuBLAS FP16 / INT8 on the same shapes.

  python tools/bench_kernels.py --suite decode|prefill|sweep|all [--out gpurun_out/kernels.jsonl]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402

L2_BYTES = 126 * 2 ** 20
LLAMA7B = [(4096, 4096), (11008, 4096), (4096, 11008)]


def kpad(k):
    return -(-k // 256) * 256


def time_graph(fn, reps, warm=3):
    s = torch.cuda.current_stream()
    for i in range(warm):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps
        best = t if best is None else min(best, t)
    return best * 1e3  # us


def tc_stages(wb, bn):
    """Mirror of gemm_tc.cu tc_stages_ct (the stage count apt_gemm validates)."""
    slots = (6 if wb <= 4 else 3) if bn <= 64 else 2
    v = ((108 if bn <= 128 else 216) * 1024 - slots * wb * 128 * 8 * 4 - (128 * (bn + 8) * 4 if bn <= 64 else 0)
         - 4096) // (bn * 128)
    return max(2, min(8, v))


def case(m, n, k, wb, ab, cfg=None, baselines=True, tag=""):
    dev = torch.device("cuda")
    wbytes = n * kpad(k) * wb // 8
    copies = max(1, min(16, -(-2 * L2_BYTES // max(wbytes, 1))))
    tiled = (cfg or {}).get("kernel", 2) != 1  # the mma.sync kernel reads canonical planes
    Ws = [P.pack(torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), dtype=torch.int8, device=dev), wb,
                 tiled=tiled) for _ in range(copies)]
    a = torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), dtype=torch.int8, device=dev)
    A = P.pack(a, ab, digits=True)
    ws = torch.rand(n, device=dev) * 1e-3
    as_ = torch.rand(m, device=dev)
    out = torch.empty((m, n), dtype=torch.float16, device=dev)
    config = cfg or P.select_config(m, n, k, wb, ab)
    wsb = P.workspace_bytes(config, m, n, k)
    work = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
    reps = max(4, min(200, int(2e5 / max(1.0, 2 * m * n * k / 1e9 * 1.0))))
    reps = 20 if m * n * k > 1e10 else (50 if m * n * k > 1e9 else 200)
    t_gemm = time_graph(lambda i: P.gemm(Ws[i % copies], A, out_kind="f16", w_scale=ws, a_scale=as_, out=out,
                                         config=config, workspace=work), reps)
    t_pack = time_graph(lambda i: P.pack(a, ab, out=A), reps)
    ops = 2 * m * n * k
    alg = wbytes + m * kpad(k) * ab // 8 + 2 * m * n + 8 * (m + n)
    row = {"tag": tag, "M": m, "N": n, "K": k, "wbits": wb, "abits": ab, "config": config,
           "gemm_us": round(t_gemm, 3), "pack_a_us": round(t_pack, 3),
           "eff_tops": round(ops / (t_gemm * 1e-6) / 1e12, 2),
           "eff_tops_incl_pack": round(ops / ((t_gemm + t_pack) * 1e-6) / 1e12, 2),
           "alg_bytes": alg, "hbm_gbs": round(alg / (t_gemm * 1e-6) / 1e9, 1), "weight_copies": copies}
    if baselines:
        wcopies = max(1, min(8, -(-2 * L2_BYTES // (2 * n * k))))
        wf = [torch.randn((n, k), device=dev, dtype=torch.float16) for _ in range(wcopies)]
        af = torch.randn((m, k), device=dev, dtype=torch.float16)
        of = torch.empty((m, n), device=dev, dtype=torch.float16)
        t16 = time_graph(lambda i: torch.matmul(af, wf[i % wcopies].t(), out=of), reps)
        del wf
        wi = [torch.randint(-8, 8, (n, k), device=dev, dtype=torch.int8) for _ in range(max(1, min(8, -(-2 * L2_BYTES // (n * k)))))]
        mi = max(m, 32)
        ai = torch.randint(-8, 8, (mi, k), device=dev, dtype=torch.int8)
        t8 = time_graph(lambda i: torch._int_mm(ai, wi[i % len(wi)].t()), reps)
        del wi
        row.update({"cublas_fp16_us": round(t16, 3), "cublas_int8_us": round(t8, 3),
                    "cublas_int8_M": mi,
                    "speedup_vs_fp16": round(t16 / t_gemm, 3), "speedup_vs_int8": round(t8 / t_gemm, 3)})
    del Ws
    torch.cuda.empty_cache()
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--suite", default="all")
    ap.add_argument("--out", default="gpurun_out/kernels.jsonl")
    ap.add_argument("--bn", type=int, default=0, help="force TC bn (128/256) for M > 64")
    ap.add_argument("--cn", type=int, default=0, help="force TC cluster_n for M > 64")
    args = ap.parse_args()
    rows = []
    cases = []
    if args.suite in ("decode", "all"):
        for m in (1, 8, 16):
            for wb, ab in ((1, 2), (2, 2), (3, 4), (4, 4)):
                for n, k in LLAMA7B:
                    cases.append(("decode", m, n, k, wb, ab))
    if args.suite in ("prefill", "all"):
        for wb, ab in ((2, 8), (4, 4)):
            for n, k in LLAMA7B:
                cases.append(("prefill", 2048, n, k, wb, ab))
    if args.suite in ("sweep", "all"):
        for wb in range(1, 9):
            for ab in range(1, 9):
                cases.append(("sweep", 4096, 4096, 4096, wb, ab))
    if args.suite in ("70b", "all"):
        for n, k in ((8192, 8192), (28672, 8192)):
            cases.append(("70b", 4096, n, k, 2, 4))
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "a") as f:
        for tag, m, n, k, wb, ab in cases:
            cfg = None
            if (args.bn or args.cn) and m > 64:
                cfg = P.select_config(m, n, k, wb, ab)
                if args.bn:
                    cfg["bn"] = args.bn
                    cfg["stages"] = tc_stages(wb, args.bn)
                if args.cn:
                    cfg["cluster_n"] = args.cn
            r = case(m, n, k, wb, ab, cfg=cfg, baselines=(tag != "sweep" or (wb, ab) in ((4, 4), (8, 8))), tag=tag)
            print(json.dumps(r), flush=True)
            f.write(json.dumps(r) + "\n")
            rows.append(r)


if __name__ == "__main__":
    main()
