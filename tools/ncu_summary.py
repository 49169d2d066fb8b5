"""Markdown summary of one `ncu --set full` capture: key throughput / traffic
metrics per captured launch plus the per-source-line stall table
(tools/ncu_stalls.py).  Usage: ncu_summary.py REPORT.ncu-rep [top_lines]."""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
top = sys.argv[2] if len(sys.argv) > 2 else "20"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
]
print(f"# ncu --set full: {os.path.basename(rep)}\n")
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print(f"## {d.get('Kernel Name', '?')[:80]} (launch id {d.get('ID')})\n")
    print("| metric | value |\n|---|---:|")
    for k, label in KEYS:
        if k in d:
            print(f"| {label} (`{k}`) | {d[k]} {u.get(k, '')} |")
    print()
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
tmp = "/tmp/_ncu_src.csv"
with open(tmp, "w") as fh:
    fh.write(src)
here = os.path.dirname(os.path.abspath(__file__))
out = subprocess.run([sys.executable, os.path.join(here, "ncu_stalls.py"), tmp, top], capture_output=True, text=True).stdout
print("## Warp-stall samples by source line\n\n```")
print(out.rstrip())
print("```")
