"""Per-unit timeline of one grouped launch (APT_LIB_VARIANT=libapt_trace.so, built with -DAPT_GRP_TRACE):
data latency (weights issued -> consumer warp 0 sees the slot full), consumer time (full -> released),
producer wait (released u - D -> weights of u issued).  usage: python tools/grp_trace.py W1A2|W4A4"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "W1A2"
PREC = {"W1A2": (1, 2), "W2A2": (2, 2), "W3A4": (3, 4), "W4A4": (4, 4)}
precs = list(PREC.values()) if which == "all" else [PREC[which]]
wb = max(p[0] for p in precs)
dev = torch.device("cuda:0")
probs = []
for (wb, ab) in precs:
  for (n, k) in [(4096, 4096), (11008, 4096), (4096, 11008)]:
    for m in (1, 8, 16):
        w = torch.randint(-(1 << (wb - 1)), 1 << (wb - 1), (n, k), dtype=torch.int8, device=dev)
        a = torch.randint(-(1 << (ab - 1)), 1 << (ab - 1), (m, k), dtype=torch.int8, device=dev)
        probs.append(dict(W=P.pack(w, wb, tiled=True), A=P.pack(a, ab, digits=True), out_kind="f16",
                          w_scale=torch.rand(n, device=dev), a_scale=torch.rand(m, device=dev)))
ws = P.grouped_workspace(dev)
L = P._lib.lib()
fn = L.apt_debug_grp_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
for _ in range(3):
    P.gemm_grouped(probs, workspace=ws)
torch.cuda.synchronize()
fn(None, 1)
torch.cuda.synchronize()
P.gemm_grouped(probs, workspace=ws)
torch.cuda.synchronize()
buf = np.zeros((1024, 128, 4), dtype=np.uint64)
fn(buf.ctypes.data, 0)
smid = buf[:, 127, 3].astype(np.int64) - 1
buf[:, 127, :] = 0
t = buf.astype(np.float64)
wb = max(p[0] for p in precs)
ctas = np.nonzero(t[:, 0, 0])[0]
t0 = t[ctas][:, :, :][t[ctas] > 0].min()
lat, comp, pw, gap = [], [], [], []
D = 4 if wb <= 2 else 2
for c in ctas:
    u_n = int(np.count_nonzero(t[c, :, 3]))
    for u in range(u_n):
        if t[c, u, 0] and t[c, u, 2]:
            lat.append(t[c, u, 2] - t[c, u, 0])
        if t[c, u, 2] and t[c, u, 3]:
            comp.append(t[c, u, 3] - t[c, u, 2])
        if u >= D and t[c, u, 0] and t[c, u - D, 3]:
            pw.append(t[c, u, 0] - t[c, u - D, 3])
        if u >= 1 and t[c, u, 2] and t[c, u - 1, 3]:
            gap.append(t[c, u, 2] - t[c, u - 1, 3])
q = lambda v: (round(float(np.percentile(v, 10)), 0), round(float(np.median(v)), 0), round(float(np.percentile(v, 90)), 0))  # noqa: E731
print(which, "ctas", len(ctas), "units/cta med", int(np.median([np.count_nonzero(t[c, :, 3]) for c in ctas])))
print("span us", round((t[ctas].max() - t0) / 1e3, 2), "first issue -> first full med ns", q([t[c, 0, 2] - t[c, 0, 0] for c in ctas]))
print("data latency issue->full ns (p10, med, p90)", q(lat))
print("consumer full->release ns", q(comp))
print("consumer idle release(u-1)->full(u) ns", q(gap))
print("producer release(u-D)->issue(u) ns", q(pw))
full_ctas = [c for c in ctas if np.count_nonzero(t[c, :, 3]) < t.shape[1]]
ends = np.array([t[c, :, 3].max() for c in full_ctas]) - t0
print("ctas with a complete trace", len(full_ctas), "end us p0/p10/p50/p90/p100",
      [round(float(np.percentile(ends, q)) / 1e3, 1) for q in (0, 10, 50, 90, 100)])
sm_end = {}
for c in full_ctas:
    sm_end[smid[c]] = max(sm_end.get(smid[c], 0), t[c, :, 3].max() - t0)
se = np.array(list(sm_end.values()))
print("SMs", len(se), "per-SM end us p0/p10/p50/p90/p100", [round(float(np.percentile(se, q)) / 1e3, 1) for q in (0, 10, 50, 90, 100)])
by_sm = {}
for c in ctas:
    by_sm.setdefault(int(smid[c]), []).append(int(c))
order = sorted(sm_end)
print("per-SM end us by smid (groups of 8):", [round(float(np.mean([sm_end[i] for i in order[j:j + 8]])) / 1e3, 1) for j in range(0, len(order), 8)])
busy_sm = {}
for c in full_ctas:
    busy_sm[int(smid[c])] = busy_sm.get(int(smid[c]), 0) + sum(
        (t[c, u, 3] - t[c, u, 2]) for u in range(t.shape[1]) if t[c, u, 3] and t[c, u, 2])
print("per-SM consumer busy (warp 0) us p0/p50/p100", [round(float(np.percentile(list(busy_sm.values()), q)) / 1e3, 1) for q in (0, 50, 100)])
print("CTAs of SM 0..3:", [by_sm.get(i) for i in range(4)], "smid of CTAs 0..9:", [int(smid[c]) for c in range(10)])
print("cta start (first issue) spread us", round((t[ctas, 0, 0].max() - t[ctas, 0, 0].min()) / 1e3, 2),
      "cta end spread us", round((max(t[c, :, 3].max() for c in ctas) - min(t[c, :, 3].max() for c in ctas)) / 1e3, 2))

# ---- per-class unit cost fit: replicate the host's stream-K split (apt.cu grp_run, same cost formula),
# count every CTA's units per (wbits, M) class, least-squares fit CTA busy time = sum_c n_c x_c
def unit_cost(wb, m):  # apt.cu grp_run
    return 4 * wb + (16 if m > 8 else 8)
meta = []  # per problem: (wb, m, units, cost)
for (pwb, pab) in precs:
    for (n, k) in [(4096, 4096), (11008, 4096), (4096, 11008)]:
        for m in (1, 8, 16):
            units = -(-n // 128) * (k // 256)
            meta.append((pwb, m, units, unit_cost(pwb, m)))
T = sum(u * c for (_, _, u, c) in meta)
cmax = max(c for (_, _, _, c) in meta)
W = min(148 * 4, T // cmax)
cls = sorted({(w, m) for (w, m, _, _) in meta})
A = np.zeros((W, len(cls)))
cost0 = 0
for (pwb, m, units, c) in meta:
    b = np.arange(units)
    owner = ((2 * cost0 + (2 * b + 1) * c) * W) // (2 * T)
    for o, cnt in zip(*np.unique(owner, return_counts=True)):
        A[o, cls.index((pwb, m))] += cnt
    cost0 += units * c
busy = np.array([t[c, :, 3].max() - t[c, 0, 0] for c in ctas[:W]])
x, *_ = np.linalg.lstsq(A[ctas[:W]] if len(ctas) >= W else A, busy, rcond=None)
print("fitted ns per unit by (wbits, M):", {f"W{k[0]} M{k[1]}": round(float(v), 1) for k, v in zip(cls, x)})
