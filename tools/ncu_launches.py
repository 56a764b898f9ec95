"""Per-kernel summary of an ncu launch list (gpu__time_duration.sum CSV): launches, total and mean
time and share of the listed GPU time, for profiles/.

  python tools/ncu_launches.py gpurun_out/launches_TAG.csv > profiles/rNN_launches.txt
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[i0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[i0 + 1:]:
    agg[r[ki].split("(")[0].strip()].append(float(r[vi].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'total_us':>10s} {'mean_us':>8s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k[:48]:48s} {len(v):8d} {sum(v):10.1f} {sum(v) / len(v):8.2f} {sum(v) / tot:6.3f}")
ours = sum(sum(v) for k, v in agg.items() if "apt::" in k or k.startswith("void gemm_tc") or "pack_kernel" in k)
print(f"# ncu per-launch times are cold-L2 and serialised; the library's kernels take {ours / tot:.3f} of the "
      f"listed time (the rest is torch's input generation / fills in bench setup)")
