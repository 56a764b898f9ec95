"""Compare decode-suite kernel times of library variants: python tools/cmp_var.py a.jsonl b.jsonl ..."""
import json
import sys

runs = [[json.loads(l) for l in open(f)] for f in sys.argv[1:]]
print("case".ljust(28) + "".join(f.split("_")[-1][:14].rjust(16) for f in sys.argv[1:]))
tot = [0.0] * len(runs)
for i, r in enumerate(runs[0]):
    name = f"M{r['M']} W{r['wbits']}A{r['abits']} {r['N']}x{r['K']}"
    ts = [run[i]["gemm_us"] for run in runs]
    for j, t in enumerate(ts):
        tot[j] += t
    print(name.ljust(28) + "".join(f"{t:16.2f}" for t in ts))
print("total".ljust(28) + "".join(f"{t:16.1f}" for t in tot))
