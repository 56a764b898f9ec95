"""Pack-kernel timings (apt_pack_bipolar): the bench step's 12 activation packs as one CUDA graph, each
activation pack alone (graph of 20 back-to-back launches), and the offline weight packs with
pre-allocated outputs (cold L2: a 256 MB write before every replay).  One JSON line per measurement.

  python tools/pack_bench.py
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_19087_b200 as P  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
g = torch.Generator(device=dev)
g.manual_seed(1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def codes(rows, k, bits):
    return torch.randint(-(1 << (bits - 1)), 1 << (bits - 1), (rows, k), generator=g, device=dev, dtype=torch.int8)


def time_graph(fn, reps=20, cold=False):
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        fn()
    for _ in range(3):
        gr.replay()
    ts = []
    for r in range(reps):
        if cold:
            flush.fill_(r & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        gr.replay()
        b.record(st)
        ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ts) * 1e3  # us


MS, ABITS, KS = [1, 8, 16], [2, 4], [4096, 11008]
acts = {(m, ab, k): codes(m, k, ab) for m in MS for ab in ABITS for k in KS}
bufs = {key: P.alloc_packed(key[0], key[2], key[1], dev, digits=True) for key in acts}


def step():
    for key, c in acts.items():
        P.pack(c, key[1], out=bufs[key])


us = time_graph(step)
print(json.dumps({"what": "act_pack_graph_12", "us": round(us, 2), "us_per_pack": round(us / 12, 3)}), flush=True)
for key, c in acts.items():
    def one(c=c, key=key):
        for _ in range(20):
            P.pack(c, key[1], out=bufs[key])
    us = time_graph(one) / 20
    print(json.dumps({"what": "act_pack_b2b", "M": key[0], "abits": key[1], "K": key[2], "us": round(us, 3)}), flush=True)

for (m, k, ab) in [(2048, 4096, 8), (2048, 4096, 4), (2048, 11008, 4), (4096, 8192, 4)]:
    c = codes(m, k, ab)
    out = P.alloc_packed(m, k, ab, dev, digits=True)
    us = time_graph(lambda: P.pack(c, ab, out=out), cold=True)
    byt = m * k + ab * m * P.kpad(k) // 8 + m * P.kpad(k) + 4 * m
    print(json.dumps({"what": "act_pack_prefill", "M": m, "K": k, "abits": ab, "us": round(us, 2),
                      "GB/s": round(byt / us / 1e3, 1)}), flush=True)
    del c, out

for (n, k) in [(4096, 4096), (11008, 4096), (4096, 11008), (8192, 8192), (28672, 8192)]:
    for wb in [1, 2, 4, 8]:
        c = codes(n, k, wb)
        out = P.alloc_packed(n, k, wb, dev, tiled=True)
        us = time_graph(lambda: P.pack(c, wb, out=out), cold=True)
        byt = n * k + wb * n * P.kpad(k) // 8 + 4 * n
        print(json.dumps({"what": "weight_pack", "N": n, "K": k, "wbits": wb, "us": round(us, 2),
                          "GB/s": round(byt / us / 1e3, 1)}), flush=True)
        del c, out
