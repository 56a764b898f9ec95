"""Tabulate tools/dec_ab.py output: one row per case, one column per config (us per launch)."""
import json
import sys
from collections import defaultdict

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
d = defaultdict(dict)
for r in rows:
    if "us" in r:
        d[(r["M"], r["N"], r["K"], r["W"], r["A"])][r["cfg"]] = r["us"]
    else:
        print("ERR", r)
cfgs = sorted({c for v in d.values() for c in v}, key=lambda c: (c != "selector", len(c), c))
print("case".ljust(26), " ".join(c.replace("dec ", "")[:8].rjust(8) for c in cfgs), "   best")
tot_sel = tot_best = 0
for k, v in sorted(d.items()):
    best = min(v, key=v.get)
    tot_sel += v.get("selector", 0)
    tot_best += v[best]
    print(str(k).ljust(26), " ".join(f"{v.get(c, float('nan')):8.2f}" for c in cfgs), "  ", best)
print("sum selector", round(tot_sel, 2), "sum best", round(tot_best, 2))
