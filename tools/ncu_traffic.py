"""DRAM traffic of the 36 decode GEMM launches of one bench.py step (ncu CSV with dram__bytes_read/
write.sum, captured with `-k regex:gemm_tc -s 72 -c 36`, i.e. one graph replay of the GEMM phase in
CASES order) -> profiles/decode_traffic.json, next to the algorithmic bytes of each case.

  python tools/ncu_traffic.py gpurun_out/traffic_TAG.csv [out.json]
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

src = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(bench.ROOT, "profiles", "decode_traffic.json")
rows = list(csv.reader(open(src)))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[i0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = {}
for r in rows[i0 + 1:]:
    d = per.setdefault(int(r[0]), {"kernel": r[ki].split("(")[0]})
    d[r[mi]] = float(r[vi].replace(",", ""))
launches = [per[k] for k in sorted(per)]
assert len(launches) == len(bench.CASES), len(launches)
cases = []
for (m, wb, ab, n, k), d in zip(bench.CASES, launches):
    alg = bench.alg_bytes(m, n, k, wb, ab)
    dram = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    cases.append({"case": f"M{m} W{wb}A{ab} {n}x{k}", "kernel": d["kernel"], "alg_bytes": alg, "dram_bytes": dram,
                  "dram_over_alg": round(dram / alg, 4), "ncu_us": d["gpu__time_duration.sum"] / 1e3})
res = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 f"(cold L2 per launch, serialised) on one bench.py GEMM phase; file {os.path.basename(src)}",
       "dram_bytes_per_launch_avg": round(sum(c["dram_bytes"] for c in cases) / len(cases)),
       "alg_bytes_per_launch_avg": round(sum(c["alg_bytes"] for c in cases) / len(cases)),
       "note": "dram writes of the fp16 outputs stay in L2 at kernel end (write-back later), so dram_bytes "
               "is essentially the packed weights + activation digits read once",
       "cases": cases}
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "cases"}, indent=1))
