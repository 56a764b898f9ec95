"""Markdown table of tools/bench_kernels.py output (one JSON object per line) for BASELINE.md.

  python tools/results_table.py gpurun_out/kern_TAG.log [title]
"""
import json
import sys

rows = []
for line in open(sys.argv[1]):
    try:
        rows.append(json.loads(line))
    except ValueError:
        pass
print("| M | N x K | W/A | config (bn, split, cluster) | APT us | eff-TOPS | HBM GB/s (alg.) | cuBLAS FP16 us | cuBLAS INT8 us | x FP16 | x INT8 |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    c = r["config"]
    print(f"| {r['M']} | {r['N']}x{r['K']} | W{r['wbits']}A{r['abits']} | {c['bn']}, {c['split_k']}, {c['cluster_n']} | "
          f"{r['gemm_us']:.2f} | {r['eff_tops']:.1f} | {r.get('hbm_gbs', 0):.0f} | {r['cublas_fp16_us']:.2f} | "
          f"{r['cublas_int8_us']:.2f} | {r['speedup_vs_fp16']:.2f} | {r['speedup_vs_int8']:.2f} |")
