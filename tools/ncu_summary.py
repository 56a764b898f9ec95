"""Summarise an ncu report: key throughput metrics and the hottest SASS lines (stall samples).

  python tools/ncu_summary.py report.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "sm__pipe_tensor_cycles_active.avg.pct", "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct", "sm__pipe_shared_cycles_active.avg.pct",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__cycles_elapsed.avg.per_second", "smsp__issue_active.avg.pct",
        "sm__inst_executed_pipe_uniform.avg.pct"]
for h, u, v in zip(hdr, units, vals):
    if any(h.startswith(w) for w in want):
        print(f"{h:80s} {u:12s} {v}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
i0 = next(i for i, r in enumerate(srows) if r and r[0] == "Address")
body = srows[i0 + 1:]
tot = sum(int(r[2]) for r in body if len(r) > 2 and r[2].isdigit())
print("samples", tot)
for r in sorted((r for r in body if len(r) > 2 and r[2].isdigit()), key=lambda r: -int(r[2]))[:top]:
    print(r[2].rjust(6), r[0][-5:], r[1][:110])
