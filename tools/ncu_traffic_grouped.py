"""DRAM traffic of the grouped decode launch(es) of one bench.py step (ncu CSV with dram__bytes_read/write.sum,
captured with `-k regex:gemm_grp -c 1` on the first eager step: one launch of the 36 problems; or `-c 4` of a
per-precision run) -> profiles/grouped_traffic.json, next to the algorithmic bytes of each launch's problems.

  python tools/ncu_traffic_grouped.py gpurun_out/traffic_grp.csv [out.json]
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

src = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(bench.ROOT, "profiles", "grouped_traffic.json")
rows = list(csv.reader(open(src)))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[i0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = {}
for r in rows[i0 + 1:]:
    d = per.setdefault(int(r[0]), {"kernel": r[ki].split("(")[0]})
    d[r[mi]] = float(r[vi].replace(",", ""))
launches = [per[k] for k in sorted(per)]
if len(launches) == 1:
    groups = [("all 36 problems", bench.CASES)]
else:
    assert len(launches) == len(bench.PRECISIONS), len(launches)
    groups = [(f"W{wb}A{ab} (9 problems)", [c for c in bench.CASES if (c[1], c[2]) == (wb, ab)]) for (wb, ab) in bench.PRECISIONS]
res_l = []
for (name, cases), d in zip(groups, launches):
    alg = sum(bench.alg_bytes(m, n, k, w, a) for (m, w, a, n, k) in cases)
    dram = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    res_l.append({"launch": name, "kernel": d["kernel"], "alg_bytes": alg, "dram_bytes": dram,
                  "dram_over_alg": round(dram / alg, 4), "ncu_us": d["gpu__time_duration.sum"] / 1e3})
res = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 f"(cold L2 per launch, serialised) on the grouped launch(es) of one bench.py step; file "
                 f"{os.path.basename(src)}",
       "dram_bytes_per_launch_avg": round(sum(c["dram_bytes"] for c in res_l) / len(res_l)),
       "alg_bytes_per_launch_avg": round(sum(c["alg_bytes"] for c in res_l) / len(res_l)),
       "launches": res_l}
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "launches"}, indent=1))
