"""The paper's ablation (§6.5) on B200: for each case, the device time of
  basic   : the paper's Basic design — p_a * p_w 1-bit x 1-bit plane-pair GEMMs (digit width 1) writing
            int32 products to HBM, then the shift-add recovery in global memory (apt_recombine_plane_products);
  fused   : the product path with full-width digits (one MMA pass, shift-add folded into the operand
            rebuild), the analytic selector's config (table cleared: the paper's step before kernel mapping);
  tuned   : the same with the autotuned table (the paper's kernel mapping, §5).
Bipolar int32 output (the paper's result) everywhere; CUDA graphs, L2 flushed before every replay.

  python tools/ablation.py > profiles/r2_ablation.jsonl
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402
from paper_2508_19087_b200 import ablation  # noqa: E402

CASES = [(16, 4096, 4096, 2, 2), (16, 11008, 4096, 4, 4), (1, 4096, 11008, 1, 2), (2048, 4096, 4096, 2, 8),
         (2048, 4096, 4096, 4, 4), (2048, 11008, 4096, 2, 2)]


def timed(fn, st, flush, reps=5):
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        fn()
    gr.replay()
    ts = []
    for r in range(reps):
        flush.fill_(r & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        gr.replay()
        b.record(st)
        ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3


def main():
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    for (m, n, k, wb, ab) in CASES:
        a = torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), generator=g, device=dev, dtype=torch.int8)
        w = torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), generator=g, device=dev, dtype=torch.int8)
        pp = ablation.PlanePairs(a, ab, w, wb)
        A = P.pack(a, ab, digits=True)
        W = P.pack(w, wb, tiled=True)
        out = torch.empty((m, n), dtype=torch.int32, device=dev)
        basic = timed(lambda: pp.basic(out=out), st, flush)
        P.clear_table()
        cfg_a = P.select_config(m, n, k, wb, ab)
        fused = timed(lambda: P.gemm(W, A, out_kind="bipolar", out=out, config=cfg_a), st, flush)
        P.load_default_table()
        cfg_t = P.select_config(m, n, k, wb, ab)
        tuned = timed(lambda: P.gemm(W, A, out_kind="bipolar", out=out, config=cfg_t), st, flush)
        ops = 2 * m * n * k
        print(json.dumps({"case": f"M{m} N{n} K{k} W{wb}A{ab}", "plane_pairs": wb * ab,
                          "basic_us": round(basic, 2), "fused_us": round(fused, 2), "tuned_us": round(tuned, 2),
                          "speedup_fused_vs_basic": round(basic / fused, 2), "speedup_tuned_vs_fused": round(fused / tuned, 3),
                          "basic_tops": round(ops / basic / 1e6, 2), "tuned_tops": round(ops / tuned / 1e6, 2),
                          "basic_hbm_recovery_bytes": 4 * m * n * (wb * ab + 1)}), flush=True)
        del pp, A, W, a, w, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
