"""Aggregate warp-stall samples per CUDA source line from
`ncu -i X --page source --csv --print-source cuda,sass` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname = None
data = []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 5 or r[1] == "Source":
        continue
    if r[0] == "-" or r[2] != "-":
        continue
    try:
        s = int(r[4])
    except ValueError:
        continue
    data.append((s, fname, r[0], r[1].strip()[:100]))
tot = sum(d[0] for d in data) or 1
for d in sorted(data, reverse=True)[:top]:
    print(f"{d[0] / tot * 100:5.1f}% {d[1]}:{d[2]} {d[3]}")
