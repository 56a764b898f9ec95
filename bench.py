#!/usr/bin/env python
"""Benchmark of the APT W_p x A_q bit-plane GEMM hot path on B200 (driver contract: one JSON line).

Default workload (BASELINE.json configs[1], "llama2-7b-decode"): one STEP is the whole per-call
hot path for every Llama-2-7B decode linear (N x K = 4096x4096, 11008x4096, 4096x11008) at
M = 1, 8, 16 tokens and W1A2, W2A2, W3A4, W4A4 (36 cases): the 12 distinct activations packed
(apt_pack_bipolar), then the 36 bit-plane GEMMs with the fused fp16 scale epilogue.  The 36 GEMMs are
independent problems; by default (--decode grouped) they run through apt_gemm_grouped, ONE persistent
launch for all 36 problems (the 12 activation packs: one apt_pack_grouped launch), every problem with its OWN packed weights (3 copies per linear,
so no problem reads another's weights from L2); --decode per_call runs 36 apt_gemm launches instead (the
per-GEMM path, also reported under `per_call` in the default run).  Weight packing is offline (done once,
timed separately and reported as `weight_pack`).  Two packed-weight sets (2 x 400 MB grouped, 2 x 133 MB
per-call, both > L2) alternate between steps so weights stream from HBM.  Steps are replayed as CUDA graphs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl apt|reference]

N > 1 (torchrun): tensor parallel N-split of every linear's weight rows, each rank computes its
[N/P, M] slice (column layout) and an NCCL all-gather assembles Y^T (strong scaling).
--impl reference: the CPU oracle (C int64 GEMM, oracle/) on host cores, rank 0 only.
"""
import argparse
import faulthandler
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective TOPS per W/A precision on Llama-7B shapes; speedup vs cuBLAS FP16/INT8"
PRECISIONS = [(1, 2), (2, 2), (3, 4), (4, 4)]            # (wbits, abits): W1A2, W2A2, W3A4, W4A4
SHAPES = [(4096, 4096), (11008, 4096), (4096, 11008)]   # (N, K) Llama-2-7B linears
MS = [1, 8, 16]
CASES = [(m, wb, ab, n, k) for m in MS for (wb, ab) in PRECISIONS for (n, k) in SHAPES]


def kpad(k):
    return -(-k // 256) * 256


def alg_bytes(m, n, k, wb, ab):
    """Algorithmic HBM bytes of one GEMM launch: packed W + packed A planes, row sums, scales, fp16 out."""
    return n * kpad(k) * wb // 8 + m * kpad(k) * ab // 8 + 8 * (m + n) + 2 * m * n


def log(msg):
    print(f"[bench] {msg}", file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="apt", choices=["apt", "reference"])
    ap.add_argument("--no-baselines", action="store_true", help="skip cuBLAS / oracle / e2e legs")
    ap.add_argument("--decode", default="grouped", choices=["grouped", "per_call"],
                    help="decode GEMM phase: apt_gemm_grouped (one launch of the 36 problems) or 36 apt_gemm launches")
    ap.add_argument("--tp-gather", default="nccl", choices=["nccl", "peer"],
                    help="N > 1, grouped decode: NCCL all-gather per output, or epilogue-direct peer stores into "
                         "symmetric-memory outputs (tp.tp_grouped_decode_peer, NEXT-4 ii)")
    ap.add_argument("--legs", default="all",
                    help="extra BASELINE configs timed in the same run: all | none | comma list of prefill,llama70b,sweep")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


KERNEL_NAMES = {2: "gemm_tc_kernel (tcgen05)", 3: "gemv_kernel (SIMT dp4a)",
                4: "gemm_skinny_kernel (mma.sync from registers)",
                5: "gemm_dec_kernel (mma.sync, weights as the streamed B operand)"}


def kernel_mix(cfgs):
    """Launch count per kernel family of one GEMM phase (from the selector's configs)."""
    mix = {}
    for c in cfgs:
        mix[KERNEL_NAMES[c["kernel"]]] = mix.get(KERNEL_NAMES[c["kernel"]], 0) + 1
    return mix


def load_traffic(name="decode_traffic.json"):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock and clock-event reasons with NVML every 50 ms in a thread."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, device_index):
        self.samples = []
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            phys = device_index
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            if vis:
                ids = [v.strip() for v in vis.split(",")]
                if device_index < len(ids) and ids[device_index].isdigit():
                    phys = int(ids[device_index])
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((time.time(), sm, rs))
            except Exception:
                pass
            time.sleep(0.05)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        if not win and self.samples:
            win = [min(self.samples, key=lambda s: abs(s[0] - (t0 + t1) / 2))]
        reasons = set()
        for _, _, rs in win:
            for bit, name in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median([s[1] for s in win]) if win else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(win)}


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    """The CPU oracle (oracle/oracle_gemm.c, int64 triple loop, OpenMP on all host cores) on the
    same workload: each step is a bounded sample, one token row of one case, rotating over the 36
    cases; same metric and unit as the GPU arm."""
    if rank != 0:
        return 0
    import numpy as np
    from oracle import c_gemm_i64, c_threads
    from synth import signed_codes
    ops_total = 0
    rng_cases = [(m, wb, ab, n, k) for (m, wb, ab, n, k) in CASES]
    data = {}
    for (m, wb, ab, n, k) in rng_cases:
        key = (wb, ab, n, k)
        if key not in data:
            data[key] = (signed_codes(1, k, ab, seed=11 * wb + ab + n), signed_codes(n, k, wb, seed=13 * wb + n + k))
    for s in range(args.warmup):
        m, wb, ab, n, k = rng_cases[s % len(rng_cases)]
        a, w = data[(wb, ab, n, k)]
        c_gemm_i64(a, w)
    t0 = time.perf_counter()
    for s in range(args.steps):
        m, wb, ab, n, k = rng_cases[s % len(rng_cases)]
        a, w = data[(wb, ab, n, k)]
        c_gemm_i64(a, w)
        ops_total += 2 * n * k
    dt = time.perf_counter() - t0
    v = ops_total / dt / 1e12
    cores = c_threads()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TOPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / max(args.steps, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": {"workload": "llama2-7b-decode",
                                            "sample": "1 token row of one linear per step, rotating over the 36 cases"},
            "cpu_baseline": {"value": v, "unit": "TOPS", "cores": cores, "kind": "oracle",
                             "sample": "1 token row x one (N,K) linear per step, rotating over 36 decode cases"},
            "e2e": {"value": v, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm

def main():
    faulthandler.enable()
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2508_19087_b200 as P

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    log("setup")
    sampler = ClockSampler(local)
    sampler.start()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    # ---- inputs (seeded, synthetic, on device): signed codes uniform over each width's range
    g = torch.Generator(device=dev)
    g.manual_seed(20250819 + 7919 * rank)

    def codes(rows, k, bits):
        lo, hi = -(1 << (bits - 1)), (1 << (bits - 1))
        return torch.randint(lo, hi, (rows, k), generator=g, device=dev, dtype=torch.int8)

    def scales(n, lo, hi):
        return torch.exp2(torch.empty(n, device=dev).uniform_(lo, hi, generator=g)).float()

    shard = {n: n // world for (n, _) in SHAPES}
    assert all(n % world == 0 for (n, _) in SHAPES)
    wbits_set = sorted({wb for wb, _ in PRECISIONS})
    W_codes, W_packed, W_scale = {}, [{}, {}], {}
    for (n, k) in SHAPES:
        for wb in wbits_set:
            for s in range(2):
                W_codes[(s, wb, n, k)] = codes(shard[n], k, wb)
            W_scale[(wb, n, k)] = scales(shard[n], -10, -6)
    A_codes = {(m, ab, k): codes(m, k, ab) for m in MS for ab in {a for _, a in PRECISIONS} for k in {k for _, k in SHAPES}}
    A_scale = {m: scales(m, -6, -2) for m in MS}
    A_buf = {key: P.alloc_packed(key[0], key[2], key[1], dev, digits=True) for key in A_codes}
    layout = "row" if world == 1 else "col"
    outs = [torch.empty((m, shard[n]) if world == 1 else (shard[n], m), dtype=torch.float16, device=dev)
            for (m, wb, ab, n, k) in CASES]
    gathered = [torch.empty((n, m), dtype=torch.float16, device=dev) if world > 1 else None
                for (m, wb, ab, n, k) in CASES]
    peer = world > 1 and args.tp_gather == "peer" and args.decode == "grouped"
    if peer:  # gathered outputs in symmetric memory: the grouped epilogue stores every rank's slice everywhere
        from paper_2508_19087_b200 import tp
        gathered, sym_h = tp.symmetric_outputs([(n, m) for (m, wb, ab, n, k) in CASES], torch.float16)
    cfgs = [P.select_config(m, shard[n], k, wb, ab) for (m, wb, ab, n, k) in CASES]

    # ---- offline weight packing (a1), timed once: outputs allocated first, one untimed pack per width
    # loads the kernels, then the 24 packs back to back between two events on the launching stream
    for wb in wbits_set:
        P.pack(codes(128, 256, wb), wb, tiled=True)
    for (s, wb, n, k), c in W_codes.items():
        W_packed[s][(wb, n, k)] = P.alloc_packed(c.shape[0], k, wb, dev, tiled=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for (s, wb, n, k), c in W_codes.items():
        P.pack(c, wb, out=W_packed[s][(wb, n, k)])
    e1.record(stream)
    barrier()
    wpack_ms = e0.elapsed_time(e1)
    wpack_bytes = sum(c.numel() + P.kpad(c.shape[1]) * c.shape[0] * wb // 8 for (s, wb, n, k), c in W_codes.items())
    del W_codes
    # grouped path: every problem has its own packed weights (the M = 1, 8, 16 problems of one launch never
    # share a weight buffer, so no problem's weights are served from L2 by another's reads), 2 sets
    W_grp = [[P.pack(codes(shard[n], k, wb), wb, tiled=True) for (m, wb, ab, n, k) in CASES] for _ in range(2)]
    PREC_IDX = [[i for i, c in enumerate(CASES) if (c[1], c[2]) == pq] for pq in PRECISIONS]
    # the step's grouped launches: all 36 problems in ONE launch (stream-K balances the mixed widths and
    # token counts; measured faster than one launch per precision, which `per_precision` times)
    STEP_GROUPS = [list(range(len(CASES)))]
    ws_grp = P.grouped_workspace(dev)

    # one step = pack every distinct activation (m, abits, K) once (12 packs; the 4096x4096 and 11008x4096
    # linears of a precision share their input), then the 36 GEMMs (+ the all-gather of each output at N>1)
    pack_problems = [dict(codes=A_codes[key], bits=key[1], out=A_buf[key]) for key in A_codes]

    def pack_step(mode=args.decode):
        if mode == "grouped":  # the 12 independent activation packs in one launch (apt_pack_grouped)
            P.pack_grouped(pack_problems, stream=stream)
            return
        for key in A_codes:
            P.pack(A_codes[key], key[1], out=A_buf[key])

    def decode_gemms(mode, wset, a_of, scale_of, out_of, gather=True, groups=None):
        """The 36 decode GEMMs of one step: apt_gemm_grouped per precision (mode "grouped"; `groups` overrides
        which problems share a launch) or one apt_gemm per case (mode "per_call"); at N > 1 each output slice
        is all-gathered."""
        if mode == "grouped":
            for idx in (STEP_GROUPS if groups is None else groups):
                if peer and gather:  # NEXT-4 ii: the GEMM's epilogue is the all-gather
                    tp.tp_grouped_decode_peer([dict(W=W_grp[wset][i], A=a_of(i), out_kind="f16",
                                                    w_scale=W_scale[CASES[i][1:2] + CASES[i][3:]], a_scale=scale_of(i))
                                               for i in idx], [gathered[i] for i in idx], [sym_h[i] for i in idx],
                                              stream=stream)
                    continue
                P.gemm_grouped([dict(W=W_grp[wset][i], A=a_of(i), out_kind="f16", layout=layout,
                                     w_scale=W_scale[CASES[i][1:2] + CASES[i][3:]], a_scale=scale_of(i),
                                     out=out_of(i)) for i in idx], workspace=ws_grp, stream=stream)
                if world > 1 and gather:
                    for i in idx:
                        dist.all_gather_into_tensor(gathered[i], out_of(i))
            return
        for i, (m, wb, ab, n, k) in enumerate(CASES):
            P.gemm(W_packed[wset][(wb, n, k)], a_of(i), out_kind="f16", layout=layout,
                   w_scale=W_scale[(wb, n, k)], a_scale=scale_of(i), out=out_of(i), config=cfgs[i])
            if world > 1 and gather:
                dist.all_gather_into_tensor(gathered[i], out_of(i))

    a_main = lambda i: A_buf[(CASES[i][0], CASES[i][2], CASES[i][4])]  # noqa: E731
    s_main = lambda i: A_scale[CASES[i][0]]  # noqa: E731
    o_main = lambda i: outs[i]  # noqa: E731

    def gemm_step(wset, mode=args.decode):
        decode_gemms(mode, wset, a_main, s_main, o_main)

    log("eager warm steps")
    for j in range(2):
        pack_step()
        gemm_step(j)
    barrier()
    use_graphs = True
    try:
        # one graph per step (12 packs + 36 GEMMs, programmatic dependent launch across the whole chain), plus
        # the two phases alone for the phase timings
        g_step, g_gemm = [], []
        for j in range(2):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=stream):
                pack_step()
                gemm_step(j)
            g_step.append(gr)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=stream):
                gemm_step(j)
            g_gemm.append(gr)
        g_pack = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_pack, stream=stream):
            pack_step()
        # the other decode path (per-call apt_gemm launches when the headline is grouped), reported beside it
        g_step_pc, g_gemm_pc = [], []
        if args.decode == "grouped":
            for j in range(2):
                gemm_step(j, "per_call")
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=stream):
                    pack_step("per_call")
                    gemm_step(j, "per_call")
                g_step_pc.append(gr)
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=stream):
                    gemm_step(j, "per_call")
                g_gemm_pc.append(gr)
    except Exception as exc:  # NCCL capture unsupported -> eager launches (still every kernel ours)
        use_graphs = False
        print(f"[bench] graph capture failed ({exc!r}); timing eager steps", file=sys.stderr)

    def run(j):
        if use_graphs:
            g_step[j % 2].replay()
        else:
            pack_step()
            gemm_step(j % 2)

    log(f"graphs={use_graphs}; warmup")
    for j in range(args.warmup):
        run(j)
    barrier()
    t_start = time.time()
    e0.record(stream)
    for j in range(args.steps):
        run(j)
    e1.record(stream)
    barrier()
    t_end = time.time()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    ops_step = sum(2 * m * n * k for (m, wb, ab, n, k) in CASES)
    value = ops_step * args.steps / (ms * 1e-3) / 1e12

    # ---- the two phases alone, right after the timed region (same clocks): the GEMM phase (36 launches,
    # weight sets alternating so weights stream from HBM) and the pack phase, CUDA events on the stream
    def phase_ms(fn_of_j, reps):
        evs = []
        for j in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn_of_j(j)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        return statistics.mean(x.elapsed_time(y) for x, y in evs[2:])
    reps = max(6, min(args.steps, 50))
    gemm_ms = phase_ms(lambda j: g_gemm[j % 2].replay() if use_graphs else gemm_step(j % 2), reps)
    pack_ms = phase_ms(lambda j: g_pack.replay() if use_graphs else pack_step(), reps)
    bytes_all = sum(alg_bytes(m, shard[n], k, wb, ab) for (m, wb, ab, n, k) in CASES)
    hbm_peak, peak_src = load_peaks()
    achieved = bytes_all / (gemm_ms * 1e-3) / 1e9
    grouped = args.decode == "grouped"
    traffic = load_traffic("grouped_traffic.json" if grouped else "decode_traffic.json")
    per_prec_pc, per_m_pc, per_kernel = breakdown(torch, P, stream, W_packed, A_buf, W_scale, A_scale, outs, cfgs, shard,
                                                  layout, use_graphs, hbm_peak)
    if grouped:
        per_prec, per_m = grouped_breakdown(torch, stream, decode_gemms, PREC_IDX, a_main, s_main, o_main, shard,
                                            use_graphs, hbm_peak)
        per_call = {"path": "12 apt_pack_bipolar + 36 apt_gemm launches per step (selector / autotuned-table configs), "
                            "the per-call weights (2 sets x 133 MB; the M = 1, 8, 16 cases of a linear share a buffer)"}
        if use_graphs:
            for j in range(args.warmup):
                g_step_pc[j % 2].replay()
            barrier()
            e0.record(stream)
            for j in range(args.steps):
                g_step_pc[j % 2].replay()
            e1.record(stream)
            barrier()
            ms_pc = e0.elapsed_time(e1) / args.steps
            gemm_ms_pc = phase_ms(lambda j: g_gemm_pc[j % 2].replay(), reps)
            ach_pc = bytes_all / (gemm_ms_pc * 1e-3) / 1e9
            per_call.update({"value": round(sum(2 * m * n * k for (m, wb, ab, n, k) in CASES) / (ms_pc * 1e-3) / 1e12, 4),
                             "unit": "TOPS", "ms_per_step": round(ms_pc, 5),
                             "gemm_us_per_step": round(1e3 * gemm_ms_pc, 2),
                             "roofline": {"bound": "hbm", "achieved": round(ach_pc, 1), "peak": hbm_peak, "unit": "GB/s",
                                          "frac": round(ach_pc / hbm_peak, 4),
                                          "traffic": (load_traffic() or {}).get("dram_bytes_per_launch_avg"),
                                          "kernel": ", ".join(f"{k} x{v}" for k, v in sorted(kernel_mix(cfgs).items())),
                                          "gemm_us_per_launch": round(1e3 * gemm_ms_pc / len(CASES), 3)}})
        per_call.update({"per_precision": per_prec_pc, "per_m": per_m_pc, "per_kernel": per_kernel})
    else:
        per_prec, per_m, per_call = per_prec_pc, per_m_pc, None
    line = {"metric": METRIC, "value": round(value, 4), "unit": "TOPS",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": {"workload": "llama2-7b-decode", "linears_NxK": SHAPES, "M": MS,
                       "precisions": [f"W{wb}A{ab}" for wb, ab in PRECISIONS], "cases_per_step": len(CASES),
                       "out": "fp16 scaled (w_scale[n], a_scale[m])",
                       "l2": ("inputs larger than L2: 2 alternating packed-weight sets (2 x 400 MB, every problem its "
                              "own weights)") if args.decode == "grouped" else
                             "inputs larger than L2: 2 alternating packed-weight sets (2 x 133 MB)",
                       "parallelism": (f"tp{world} (N-split + " + ("epilogue-direct peer stores" if peer else "NCCL all-gather")
                                       + ")") if world > 1 else "single GPU",
                       "cuda_graphs": use_graphs},
            "gpu_launches": ((1 + len(STEP_GROUPS)) if grouped else (len(A_codes) + len(CASES))) * args.steps,
            "decode_path": ("apt_gemm_grouped: one persistent launch of the 36 independent problems (every problem "
                            "its own packed weights)") if grouped else "36 apt_gemm launches",
            "roofline": {"bound": "hbm",
                         "kernel": ("gemm_grp_kernel (apt_gemm_grouped) x1 launch/step" if grouped else
                                    "decode GEMM phase: " + ", ".join(
                                        f"{k} x{v}" for k, v in sorted(kernel_mix(cfgs).items())) + " launches/step"),
                         "measured": "GEMM phase replayed alone right after the timed region (events around the graph "
                                     "of the step's GEMM launches" + (" + all-gathers" if world > 1 else "") +
                                     ", the two weight sets alternating)",
                         "achieved": round(achieved, 1), "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4),
                         "traffic": traffic.get("dram_bytes_per_launch_avg") if traffic else None,
                         "traffic_source": (traffic or {}).get("source"),
                         "alg_bytes_per_launch_avg": round(bytes_all / (len(STEP_GROUPS) if grouped else len(CASES))),
                         "gemm_share_of_step": round(gemm_ms / ms_per_step, 3),
                         "gemm_us_per_launch": round(1e3 * gemm_ms / (len(STEP_GROUPS) if grouped else len(CASES)), 3)},
            "act_pack": {"launches_per_step": 1 if grouped else len(A_codes), "packs_per_step": len(A_codes),
                         "us_per_step": round(1e3 * pack_ms, 3),
                         "path": "apt_pack_grouped (12 packs, one launch)" if grouped else "12 apt_pack_bipolar"},
            "per_precision": per_prec, "per_m": per_m,
            **({"per_call": per_call} if grouped else {"per_kernel": per_kernel}),
            "weight_pack": {"ms": round(wpack_ms, 3), "GB/s": round(wpack_bytes / (wpack_ms * 1e-3) / 1e9, 1)}}

    legs = {"prefill", "llama70b", "sweep"} if args.legs == "all" else set() if args.legs == "none" else \
        set(args.legs.split(","))
    if legs:
        log(f"legs {sorted(legs)}")
        line.update(run_legs(args, torch, P, dev, stream, world, rank, barrier, legs))
    log("baselines")
    if not args.no_baselines:
        line.update(baselines(args, P, dev, stream, world, rank, shard, W_packed, W_scale, A_scale, cfgs, layout,
                              value, barrier, decode_gemms, (per_call or {}).get("value")))
    clocks = sampler.summary(t_start, t_end)
    sampler.stop()
    line["clocks"] = clocks
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- BASELINE configs[2]-[4] legs

def _chain_us(torch, stream, fn, n_launch, reps, flush):
    """Device time per launch of a CUDA graph of fn() (n_launch GEMMs), L2 flushed (256 MB write) before
    every replay, CUDA events on the launching stream around the replay only; median over reps."""
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=stream):
        fn()
    gr.replay()
    ts = []
    for r in range(reps):
        flush.fill_(r & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        gr.replay()
        b.record(stream)
        ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3 / n_launch


def _int8_peak(torch, dev):
    """Measured dense int8 tensor peak: cuBLAS INT8 (torch._int_mm) 8192^3, best of 10 (burst)."""
    a = torch.randint(-8, 8, (8192, 8192), device=dev, dtype=torch.int8)
    b = torch.randint(-8, 8, (8192, 8192), device=dev, dtype=torch.int8).t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2 * 8192 ** 3 / (best * 1e-3) / 1e12


def run_legs(args, torch, P, dev, stream, world, rank, barrier, legs):
    """configs[2] (Llama-2-7B prefill, M = 2048, W2A8 / W4A4, next to cuBLAS INT8 / FP16), configs[3]
    (Llama-3-70B linears, M = 4096, W2A4, N-split over the ranks: GEMM only and GEMM + all-gather, with the
    NVLink ingress bound) and configs[4] (4096^3 for all 64 (p_w, p_a)), every GEMM in the selector's
    config (autotuned table), fp16 epilogue with per-channel and per-token scales.  Tensor-bound: roofline =
    achieved TOPS / the measured int8 peak (cuBLAS _int_mm 8192^3, this run; x2 nominal for kind::mxf4)."""
    out = {}
    g = torch.Generator(device=dev)
    g.manual_seed(424242 + rank)
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
    peak = _int8_peak(torch, dev)
    out["int8_peak"] = {"TOPS": round(peak, 1), "how": "cuBLAS INT8 torch._int_mm 8192^3, best of 10 (burst), this run"}

    def codes(rows, k, bits):
        return torch.randint(-(1 << (bits - 1)), 1 << (bits - 1), (rows, k), generator=g, device=dev, dtype=torch.int8)

    def scales(n, lo, hi):
        return torch.exp2(torch.empty(n, device=dev).uniform_(lo, hi, generator=g)).float()

    def ours(m, n, k, wb, ab, copies=2):
        Ws = [P.pack(codes(n, k, wb), wb, tiled=True) for _ in range(copies)]
        a_codes = codes(m, k, ab)
        A = P.pack(a_codes, ab, digits=True)
        wsc, asc = scales(n, -10, -6), scales(m, -6, -2)
        o = torch.empty((m, n), dtype=torch.float16, device=dev)
        cfg = P.select_config(m, n, k, wb, ab)

        def fn():
            for W in Ws:
                P.gemm(W, A, out_kind="f16", w_scale=wsc, a_scale=asc, out=o, config=cfg)
        us = _chain_us(torch, stream, fn, len(Ws), 5, flush)
        pack_us = _chain_us(torch, stream, lambda: P.pack(a_codes, ab, out=A), 1, 5, flush)
        del Ws
        return us, pack_us, cfg

    if "prefill" in legs and world == 1:
        rows = []
        for (wb, ab) in ((2, 8), (4, 4)):
            for (n, k) in SHAPES:
                m = 2048
                us, pack_us, cfg = ours(m, n, k, wb, ab)
                ops = 2 * m * n * k
                a8 = torch.randint(-8, 8, (m, k), device=dev, dtype=torch.int8)
                w8 = torch.randint(-8, 8, (n, k), device=dev, dtype=torch.int8)
                int8_us = _chain_us(torch, stream, lambda: torch._int_mm(a8, w8.t()), 1, 5, flush)
                a16 = torch.randn((m, k), device=dev, dtype=torch.float16)
                w16 = torch.randn((n, k), device=dev, dtype=torch.float16)
                fp16_us = _chain_us(torch, stream, lambda: torch.matmul(a16, w16.t()), 1, 5, flush)
                del a8, w8, a16, w16
                tops = ops / us / 1e6
                mx = cfg["mma_kind"] == 1
                rows.append({"case": f"M{m} N{n} K{k} W{wb}A{ab}", "us": round(us, 2), "eff_tops": round(tops, 1),
                             "act_pack_us": round(pack_us, 2), "tops_incl_pack": round(ops / (us + pack_us) / 1e6, 1),
                             "cublas_int8_us": round(int8_us, 2), "cublas_fp16_us": round(fp16_us, 2),
                             "speedup_vs_int8": round(int8_us / us, 3), "speedup_vs_fp16": round(fp16_us / us, 3),
                             "tensor_frac": round(tops / (peak * (2 if mx else 1)), 4),
                             "kernel": ("persistent " if cfg["kernel"] == 6 else "") +
                                       ("tcgen05 kind::mxf4" if mx else "tcgen05 kind::i8"), "bn": cfg["bn"]})
        tot_ops = sum(2 * 2048 * n * k for _ in range(2) for (n, k) in SHAPES)
        tot_us = sum(r["us"] for r in rows)
        out["prefill"] = {"workload": "BASELINE configs[2]: Llama-2-7B prefill M=2048, W2A8 and W4A4",
                          "eff_tops": round(tot_ops / tot_us / 1e6, 1),
                          "speedup_vs_int8": round(sum(r["cublas_int8_us"] for r in rows) / tot_us, 3),
                          "speedup_vs_fp16": round(sum(r["cublas_fp16_us"] for r in rows) / tot_us, 3),
                          "timing": "2 packed-weight copies chained per CUDA graph, 256 MB L2 flush before each replay",
                          "cases": rows}

    if "llama70b" in legs:
        rows = []
        m, k, wb, ab = 4096, 8192, 2, 4
        for n_total in (8192, 28672):
            n = n_total // world
            us, pack_us, cfg = ours(m, n, k, wb, ab, copies=2)
            gather_us = None
            if world > 1:
                import torch.distributed as dist
                from paper_2508_19087_b200 import tp
                chunks = 4
                W = P.pack(codes(n, k, wb), wb, tiled=True)
                A = [P.pack(codes(m // chunks, k, ab), ab, digits=True) for _ in range(chunks)]
                wsc, asc = scales(n, -10, -6), scales(m, -6, -2)
                yt = torch.empty((chunks, n_total, m // chunks), dtype=torch.float16, device=dev)
                for _ in range(2):
                    tp.tp_gemm(W, A, n_total, out_kind="f16", w_scale_local=wsc, a_scale=asc, m_chunks=chunks, out=yt)
                barrier()
                ts = []
                for r in range(5):
                    flush.fill_(r & 255)
                    barrier()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    tp.tp_gemm(W, A, n_total, out_kind="f16", w_scale_local=wsc, a_scale=asc, m_chunks=chunks, out=yt)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
                t = torch.tensor([statistics.median(ts), us], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                gather_us, us = float(t[0]), float(t[1])
                del W, A, yt
            ops = 2 * m * n_total * k
            ingress_us = (world - 1) / world * 2 * m * n_total / 770e9 * 1e6 if world > 1 else None
            rows.append({"case": f"M{m} N{n_total} K{k} W{wb}A{ab}", "n_per_rank": n,
                         "gemm_us": round(us, 2), "gemm_eff_tops": round(ops / us / 1e6, 1),
                         "gemm_tensor_frac_per_gpu": round(ops / world / us / 1e6 / peak, 4),
                         "gemm_gather_us": round(gather_us, 2) if gather_us else None,
                         "gemm_gather_eff_tops": round(ops / gather_us / 1e6, 1) if gather_us else None,
                         "ingress_bound_us": round(ingress_us, 1) if ingress_us else None,
                         "kernel": ("persistent " if cfg["kernel"] == 6 else "") +
                                   ("tcgen05 kind::mxf4" if cfg["mma_kind"] == 1 else "tcgen05 kind::i8")})
        out["llama70b_tp"] = {"workload": f"BASELINE configs[3]: Llama-3-70B linears M=4096 W2A4, N-split over {world} "
                                          "GPU(s), column-layout slices, NCCL all-gather of 4 M-chunks overlapped "
                                          "with the next chunk's GEMM (N>1)",
                              "ingress": "(P-1)/P x 2 M N bytes at the measured 770 GB/s per direction (B200_PROFILING)",
                              "timing": "device time, max over ranks", "cases": rows}

    if "sweep" in legs and world == 1:
        n = m = k = 4096
        Ws = {wb: [P.pack(codes(n, k, wb), wb, tiled=True) for _ in range(2)] for wb in range(1, 9)}
        As = {ab: P.pack(codes(m, k, ab), ab, digits=True) for ab in range(1, 9)}
        wsc, asc = scales(n, -10, -6), scales(m, -6, -2)
        o = torch.empty((m, n), dtype=torch.float16, device=dev)
        res, kinds = {}, {}
        for wb in range(1, 9):
            for ab in range(1, 9):
                cfg = P.select_config(m, n, k, wb, ab)

                def fn(wb=wb, ab=ab, cfg=cfg):
                    for W in Ws[wb]:
                        P.gemm(W, As[ab], out_kind="f16", w_scale=wsc, a_scale=asc, out=o, config=cfg)
                us = _chain_us(torch, stream, fn, 2, 3, flush)
                res[f"W{wb}A{ab}"] = round(2 * m * n * k / us / 1e6, 1)
                kinds[f"W{wb}A{ab}"] = ("mxf4" if cfg["mma_kind"] == 1 else "i8") + f"/bn{cfg['bn']}"
        vals = list(res.values())
        out["sweep"] = {"workload": "BASELINE configs[4]: 4096^3, W1-W8 x A1-A8, selector (autotuned table) config",
                        "eff_tops": res, "config": kinds, "min_tops": min(vals), "max_tops": max(vals),
                        "tensor_frac_max": round(max(vals) / peak, 4),
                        "timing": "2 packed-weight copies chained per CUDA graph, L2 flushed before each replay"}
        del Ws, As
    del flush
    return out


def breakdown(torch, P, stream, W_packed, A_buf, W_scale, A_scale, outs, cfgs, shard, layout, use_graphs, hbm_peak):
    """GEMM-only throughput per precision and per M (outside the timed region): a graph of that group's
    GEMMs (packed activations resident), replayed 10x per weight set with a 256 MB write between
    replays so every replay streams its weights from HBM; events around each replay."""
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=stream.device)

    def group_stats(idx):
        gs = []
        for wset in range(2):
            def fn():
                for i in idx:
                    m, wb, ab, n, k = CASES[i]
                    P.gemm(W_packed[wset][(wb, n, k)], A_buf[(m, ab, k)], out_kind="f16", layout=layout,
                           w_scale=W_scale[(wb, n, k)], a_scale=A_scale[m], out=outs[i], config=cfgs[i])
            fn()
            if use_graphs:
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=stream):
                    fn()
                gs.append(gr.replay)
            else:
                gs.append(fn)
        ts = []
        for r in range(20):
            flush.fill_(r & 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            gs[r % 2]()
            b.record(stream)
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(x.elapsed_time(y) for x, y in ts)
        ops = sum(2 * CASES[i][0] * shard[CASES[i][3]] * CASES[i][4] for i in idx)
        byt = sum(alg_bytes(CASES[i][0], shard[CASES[i][3]], CASES[i][4], CASES[i][1], CASES[i][2]) for i in idx)
        return {"gemm_us_avg": round(1e3 * ms / len(idx), 2), "eff_tops": round(ops / (ms * 1e-3) / 1e12, 3),
                "hbm_frac": round(byt / (ms * 1e-3) / 1e9 / hbm_peak, 4)}

    per_prec = {f"W{wb}A{ab}": group_stats([i for i, c in enumerate(CASES) if c[1] == wb and c[2] == ab])
                for (wb, ab) in PRECISIONS}
    per_m = {f"M{m}": group_stats([i for i, c in enumerate(CASES) if c[0] == m]) for m in MS}
    # per kernel family (the selector's choice per case): each family's own HBM roofline fraction
    fams = sorted({c["kernel"] for c in cfgs})
    per_kernel = {KERNEL_NAMES[f]: dict(group_stats([i for i, c in enumerate(cfgs) if c["kernel"] == f]),
                                        launches=sum(1 for c in cfgs if c["kernel"] == f)) for f in fams}
    del flush
    return per_prec, per_m, per_kernel


def grouped_breakdown(torch, stream, decode_gemms, prec_idx, a_of, s_of, o_of, shard, use_graphs, hbm_peak):
    """Grouped path per precision (its own single apt_gemm_grouped launch of 9 problems) and per M (one launch
    of that M's 12 problems, mixed widths): graph replays with a 256 MB write between them, events around each."""
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=stream.device)
    import paper_2508_19087_b200 as P

    def stats(idx, decode_one):
        gs = []
        for wset in range(2):
            fn = (lambda w=wset: decode_one(w))
            fn()
            if use_graphs:
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=stream):
                    fn()
                gs.append(gr.replay)
            else:
                gs.append(fn)
        ts = []
        for r in range(20):
            flush.fill_(r & 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            gs[r % 2]()
            b.record(stream)
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(x.elapsed_time(y) for x, y in ts)
        ops = sum(2 * CASES[i][0] * shard[CASES[i][3]] * CASES[i][4] for i in idx)
        byt = sum(alg_bytes(CASES[i][0], shard[CASES[i][3]], CASES[i][4], CASES[i][1], CASES[i][2]) for i in idx)
        return {"launch_us": round(1e3 * ms, 2), "problems": len(idx), "eff_tops": round(ops / (ms * 1e-3) / 1e12, 3),
                "hbm_frac": round(byt / (ms * 1e-3) / 1e9 / hbm_peak, 4)}

    def one_launch(idx):
        return lambda wset: decode_gemms("grouped", wset, a_of, s_of, o_of, gather=False, groups=[idx])

    per_prec = {f"W{wb}A{ab}": stats(idx, one_launch(idx)) for (wb, ab), idx in zip(PRECISIONS, prec_idx)}
    per_m = {f"M{m}": stats([i for i, c in enumerate(CASES) if c[0] == m],
                            one_launch([i for i, c in enumerate(CASES) if c[0] == m])) for m in MS}
    del flush
    return per_prec, per_m


def baselines(args, P, dev, stream, world, rank, shard, W_packed, W_scale, A_scale, cfgs, layout, value, barrier,
              decode_gemms, per_call_value=None):
    """e2e through the public API with host buffers; cuBLAS FP16 / INT8 on the same cases; the CPU
    oracle on a bounded sample (rank 0, N=1)."""
    import torch
    res = {}
    # ---- e2e: pinned host activations -> device, (quantize +) pack, GEMM, fp16 result -> pinned host.
    # One pinned staging buffer each way, so a step is 1 H2D copy, 12 packs, 36 GEMMs, 1 D2H copy.
    # "e2e" (the headline): fp16 activations through apt_quantize_pack (per-token scale = the GEMM's
    # a_scale) -- what a quantized linear layer is fed; "e2e_codes": int8 codes through apt_pack_bipolar.
    keys = []
    for (m, wb, ab, n, k) in CASES:
        if (m, ab, k) not in keys:
            keys.append((m, ab, k))
    a_off, off = {}, 0
    for key in keys:
        a_off[key] = off
        off += key[0] * key[2]
    o_shapes = [(m, shard[n]) if world == 1 else (shard[n], m) for (m, wb, ab, n, k) in CASES]
    o_total = sum(a * b for a, b in o_shapes)
    d_out_all = torch.empty(o_total, dtype=torch.float16, device=dev)
    h_out_all = torch.empty(o_total, dtype=torch.float16).pin_memory()
    d_out, o = [], 0
    for (a, b) in o_shapes:
        d_out.append(d_out_all[o:o + a * b].view(a, b))
        o += a * b
    ops_step = sum(2 * m * n * k for (m, wb, ab, n, k) in CASES)
    bufs = {key: P.alloc_packed(key[0], key[2], key[1], dev, digits=True) for key in keys}
    q_scale = {key: torch.empty(key[0], dtype=torch.float32, device=dev) for key in keys}

    def e2e_packs(d_a, fp16):
        """The step's 12 activation packs (quantize + pack from fp16, or pack from int8 codes): one
        apt_pack_grouped launch on the grouped path, 12 single calls on the per-call path."""
        if args.decode == "grouped":
            P.pack_grouped([dict(x=d_a[key], bits=key[1], out=bufs[key], scale=q_scale[key]) if fp16 else
                            dict(codes=d_a[key], bits=key[1], out=bufs[key]) for key in keys], stream=stream)
            return
        for key in keys:
            if fp16:
                P.quantize_pack(d_a[key], key[1], out=bufs[key], scale=q_scale[key])
            else:
                P.pack(d_a[key], key[1], out=bufs[key])

    def e2e_leg(fp16):
        if fp16:
            h_in = torch.empty(off, dtype=torch.float16).pin_memory()
            h_in.copy_(torch.randn(off, dtype=torch.float32).to(torch.float16))
        else:
            h_in = torch.empty(off, dtype=torch.int8).pin_memory()
            for key in keys:
                m, ab, k = key
                lo, hi = -(1 << (ab - 1)), (1 << (ab - 1))
                h_in[a_off[key]:a_off[key] + m * k].copy_(torch.randint(lo, hi, (m * k,), dtype=torch.int8))
        d_in = torch.empty(off, dtype=h_in.dtype, device=dev)
        d_a = {key: d_in[a_off[key]:a_off[key] + key[0] * key[2]].view(key[0], key[2]) for key in keys}

        def e2e_step(wset):
            d_in.copy_(h_in, non_blocking=True)
            e2e_packs(d_a, fp16)
            decode_gemms(args.decode, wset, lambda i: bufs[(CASES[i][0], CASES[i][2], CASES[i][4])],
                         lambda i: q_scale[(CASES[i][0], CASES[i][2], CASES[i][4])] if fp16 else A_scale[CASES[i][0]],
                         lambda i: d_out[i], gather=False)
            h_out_all.copy_(d_out_all, non_blocking=True)

        n_e2e = max(2, min(args.steps, 50))
        graphs = []
        try:
            for j in range(2):
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=stream):
                    e2e_step(j)
                graphs.append(gr)
            run = lambda j: graphs[j % 2].replay()  # noqa: E731
        except Exception:
            run = lambda j: e2e_step(j % 2)  # noqa: E731
        for j in range(3):
            run(j)
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for j in range(n_e2e):
            run(j)
        s1.record()
        barrier()
        e2e_ms = s0.elapsed_time(s1) / n_e2e
        gm = "1x apt_gemm_grouped (36 GEMMs, fp16)" if args.decode == "grouped" else "36x apt_gemm (fp16)"
        qp = "apt_pack_grouped (12 quantize + packs)" if args.decode == "grouped" else "12x apt_quantize_pack"
        pp = "apt_pack_grouped (12 packs)" if args.decode == "grouped" else "12x apt_pack_bipolar"
        path = (f"pinned host fp16 activations -> 1 H2D -> {qp} -> {gm} -> 1 D2H"
                if fp16 else f"pinned host int8 codes -> 1 H2D -> {pp} -> {gm} -> 1 D2H")
        return {"value": round(ops_step / (e2e_ms * 1e-3) / 1e12, 4), "unit": "TOPS",
                "h2d_bytes_per_step": h_in.numel() * h_in.element_size(), "d2h_bytes_per_step": o_total * 2,
                "ms_per_step": round(e2e_ms, 5), "steps": n_e2e, "path": path + ", CUDA graph"}

    def e2e_pipelined(fp16):
        """The same end-to-end step as a serving loop runs it: step j's H2D copy (stream 1), its 12 packs +
        36 GEMMs (stream 2, CUDA graph) and its D2H copy of all fp16 results (stream 3) on double-buffered
        pinned host / device buffers, ordered by events, so step j+1's upload and compute overlap step j's
        download.  Every step still moves its own inputs up and its own results down inside the timed region
        (first H2D start to last D2H end)."""
        dt = torch.float16 if fp16 else torch.int8
        h_in = [torch.empty(off, dtype=dt).pin_memory() for _ in range(2)]
        for h in h_in:
            if fp16:
                h.copy_(torch.randn(off, dtype=torch.float32).to(torch.float16))
            else:
                for key in keys:
                    m, ab, k = key
                    lo, hi = -(1 << (ab - 1)), (1 << (ab - 1))
                    h[a_off[key]:a_off[key] + m * k].copy_(torch.randint(lo, hi, (m * k,), dtype=torch.int8))
        d_in = [torch.empty(off, dtype=dt, device=dev) for _ in range(2)]
        d_o = [torch.empty(o_total, dtype=torch.float16, device=dev) for _ in range(2)]
        h_o = [torch.empty(o_total, dtype=torch.float16).pin_memory() for _ in range(2)]
        s_up, s_dn = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        graphs = []
        for b in range(2):
            d_a = {key: d_in[b][a_off[key]:a_off[key] + key[0] * key[2]].view(key[0], key[2]) for key in keys}
            outs_b, o2 = [], 0
            for (a_, b_) in o_shapes:
                outs_b.append(d_o[b][o2:o2 + a_ * b_].view(a_, b_))
                o2 += a_ * b_

            def comp(b=b, d_a=d_a, outs_b=outs_b):
                e2e_packs(d_a, fp16)
                decode_gemms(args.decode, b, lambda i: bufs[(CASES[i][0], CASES[i][2], CASES[i][4])],
                             lambda i: q_scale[(CASES[i][0], CASES[i][2], CASES[i][4])] if fp16 else A_scale[CASES[i][0]],
                             lambda i: outs_b[i], gather=False)
            comp()
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=stream):
                comp()
            graphs.append(gr)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_comp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        ev_free = [torch.cuda.Event() for _ in range(2)]  # compute finished reading d_in[b]
        for b in range(2):  # all buffers start free
            ev_out[b].record(s_dn)
            ev_free[b].record(stream)

        def step(j):
            b = j % 2
            s_up.wait_event(ev_free[b])
            with torch.cuda.stream(s_up):
                d_in[b].copy_(h_in[b], non_blocking=True)
            ev_in[b].record(s_up)
            stream.wait_event(ev_in[b])
            stream.wait_event(ev_out[b])
            graphs[b].replay()
            ev_comp[b].record(stream)
            ev_free[b].record(stream)
            s_dn.wait_event(ev_comp[b])
            with torch.cuda.stream(s_dn):
                h_o[b].copy_(d_o[b], non_blocking=True)
            ev_out[b].record(s_dn)

        n_e2e = max(4, min(args.steps, 50))
        for j in range(4):
            step(j)
        torch.cuda.synchronize()
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(s_up)
        stream.wait_event(s0)
        s_dn.wait_event(s0)
        for j in range(n_e2e):
            step(j)
        s1.record(s_dn)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = s0.elapsed_time(s1) / n_e2e
        gm = "1x apt_gemm_grouped (36 GEMMs, fp16)" if args.decode == "grouped" else "36x apt_gemm (fp16)"
        qp = "apt_pack_grouped (12 quantize + packs)" if args.decode == "grouped" else "12x apt_quantize_pack"
        pp = "apt_pack_grouped (12 packs)" if args.decode == "grouped" else "12x apt_pack_bipolar"
        path = (f"pinned host fp16 activations -> H2D -> {qp} -> {gm} -> D2H" if fp16
                else f"pinned host int8 codes -> H2D -> {pp} -> {gm} -> D2H")
        return {"value": round(ops_step / (e2e_ms * 1e-3) / 1e12, 4), "unit": "TOPS",
                "h2d_bytes_per_step": off * (2 if fp16 else 1), "d2h_bytes_per_step": o_total * 2,
                "ms_per_step": round(e2e_ms, 5), "steps": n_e2e,
                "path": path + "; copies on their own streams, double-buffered, step j+1's upload and compute "
                               "overlapping step j's download (CUDA graph per buffer)"}

    res["e2e"] = e2e_pipelined(True)
    res["e2e_codes"] = e2e_pipelined(False)
    res["e2e_serial"] = e2e_leg(True)
    n_e2e = res["e2e"]["steps"]

    # ---- cuBLAS FP16 and INT8 on the same 36 cases (dense weights, 2 alternating sets)
    if world == 1:
        try:
            wf = [{(n, k): torch.randn((n, k), device=dev, dtype=torch.float16) for (n, k) in SHAPES} for _ in range(2)]
            af = {(m, k): torch.randn((m, k), device=dev, dtype=torch.float16) for m in MS for (_, k) in SHAPES}
            cf = [[torch.empty((m, n), device=dev, dtype=torch.float16) for (m, wb, ab, n, k) in CASES] for _ in range(2)]

            def fp16_step(s):
                for i, (m, wb, ab, n, k) in enumerate(CASES):
                    torch.matmul(af[(m, k)], wf[s][(n, k)].t(), out=cf[s][i])
            res["cublas_fp16"] = _time_graph_pair(torch, stream, fp16_step, n_e2e, ops_step, barrier)
            del wf
            wi = [{(n, k): torch.randint(-8, 8, (n, k), device=dev, dtype=torch.int8) for (n, k) in SHAPES}
                  for _ in range(2)]
            ai = {(m, k): torch.randint(-8, 8, (32, k), device=dev, dtype=torch.int8) for m in MS for (_, k) in SHAPES}

            def int8_step(s):
                for i, (m, wb, ab, n, k) in enumerate(CASES):
                    torch._int_mm(ai[(m, k)], wi[s][(n, k)].t())
            r = _time_graph_pair(torch, stream, int8_step, n_e2e, ops_step, barrier)
            r["note"] = "torch._int_mm needs M > 16: activations padded to 32 rows; ops counted at the true M"
            res["cublas_int8"] = r
            del wi
            res["speedup_vs_cublas_fp16"] = round(value / res["cublas_fp16"]["value"], 3)
            res["speedup_vs_cublas_int8"] = round(value / res["cublas_int8"]["value"], 3)
            res["cublas_note"] = ("cuBLAS runs the 36 GEMMs as 36 launches (torch exposes no grouped GEMM for mixed "
                                  "shapes); the like-for-like per-launch ratio is per_call_speedup_*")
            if per_call_value:
                res["per_call_speedup_vs_cublas_fp16"] = round(per_call_value / res["cublas_fp16"]["value"], 3)
                res["per_call_speedup_vs_cublas_int8"] = round(per_call_value / res["cublas_int8"]["value"], 3)
        except Exception as exc:
            res["cublas_error"] = repr(exc)

    # ---- CPU oracle on a bounded sample (rank 0, N=1 only)
    if rank == 0 and world == 1:
        try:
            from oracle import c_gemm_i64, c_threads
            import numpy as np
            samples = []
            for (wb, ab) in PRECISIONS:
                for (n, k) in SHAPES:
                    lo, hi = -(1 << (ab - 1)), (1 << (ab - 1))
                    a = np.random.default_rng(n + k + ab).integers(lo, hi, size=(1, k)).astype(np.int8)
                    w = np.random.default_rng(n * k + wb).integers(-(1 << (wb - 1)), 1 << (wb - 1),
                                                                    size=(n, k)).astype(np.int8)
                    samples.append((a, w))
            # repeat the 36-case sample (one token row per case) until >= 10 s of CPU work
            t0 = time.perf_counter()
            ops = 0
            reps = 0
            while time.perf_counter() - t0 < 10.0:
                for rep in range(len(MS)):
                    for a, w in samples:
                        c_gemm_i64(a, w)
                        ops += 2 * w.shape[0] * w.shape[1]
                reps += 1
            dt = time.perf_counter() - t0
            res["cpu_baseline"] = {"value": round(ops / dt / 1e12, 6), "unit": "TOPS", "cores": c_threads(),
                                   "kind": "oracle",
                                   "sample": "1 token row for each of the 36 decode cases (12 (precision, linear) "
                                             "pairs x 3), C int64 triple loop, OpenMP, repeated for >= 10 s",
                                   "seconds": round(dt, 3), "passes": reps}
        except Exception as exc:
            res["cpu_baseline"] = {"error": repr(exc)}
    return res


def _time_graph_pair(torch, stream, fn, n, ops_step, barrier):
    graphs = []
    fn(0)
    fn(1)
    barrier()
    for j in range(2):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            fn(j)
        graphs.append(gr)
    for j in range(3):
        graphs[j % 2].replay()
    barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for j in range(n):
        graphs[j % 2].replay()
    s1.record()
    barrier()
    ms = s0.elapsed_time(s1) / n
    return {"value": round(ops_step / (ms * 1e-3) / 1e12, 4), "unit": "TOPS", "ms_per_step": round(ms, 5)}


if __name__ == "__main__":
    sys.exit(main())
