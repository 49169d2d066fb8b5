"""Per-source-line stall breakdown from
`ncu -i X --page source --csv --print-source cuda,sass` output:
prints the top lines by samples with their dominant stall reasons, and the
kernel-wide stall totals."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
fname = None
tot = defaultdict(float)
lines = []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr) or r[0] == "-" or r[2] != "-":
        continue
    d = dict(zip(hdr[4:], r[4:]))
    st = {}
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                st[k[6:]] = float(v)
            except ValueError:
                pass
    for k, v in st.items():
        tot[k] += v
    s = sum(st.values())
    lines.append((s, f"{fname}:{r[0]}", r[1].strip()[:70], st))
T = sum(tot.values()) or 1
print("kernel stalls:", ", ".join(f"{k} {v / T * 100:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
for s, loc, src, st in sorted(lines, key=lambda x: -x[0])[:top]:
    dom = ", ".join(f"{k} {v / max(s, 1) * 100:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{s / T * 100:5.1f}% {loc} [{dom}] {src}")
