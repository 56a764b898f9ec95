"""Compare bench_kernels decode logs of several variants: python tools/cmp_kern.py TAG v1 v2 ..."""
import json
import sys

tag, vs = sys.argv[1], sys.argv[2:]


def load(f):
    d = {}
    for line in open(f):
        try:
            r = json.loads(line)
        except ValueError:
            continue
        d[(r['M'], r['N'], r['K'], r['wbits'], r['abits'])] = r['gemm_us']
    return d


D = {v: load(f'gpurun_out/kern_{tag}_{v}.log') for v in vs}
print(' '.join(vs))
tot = {v: 0.0 for v in vs}
for k in D[vs[0]]:
    print(k, *[D[v].get(k) for v in vs])
    for v in vs:
        tot[v] += D[v].get(k, 0)
print({v: round(t, 2) for v, t in tot.items()})
