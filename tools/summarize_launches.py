"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) of
`bench.py --steps 1`: per-kernel launch count, device time and share of the
last step (launches from the last k_assemble on).  ncu serialises launches and
runs them cold, so shares, not absolute times, are comparable with bench.py."""
import csv
import re
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
names = [re.sub(r"\(.*", "", r[4]).replace("void ", "") for r in rows]
times = [float(r[14]) for r in rows]
start = max(i for i, n in enumerate(names) if n.startswith("k_assemble"))
agg = OrderedDict()
for n, t in zip(names[start:], times[start:]):
    c, s = agg.get(n, (0, 0.0))
    agg[n] = (c + 1, s + t)
tot = sum(s for _, s in agg.values())
print(f"launches in the last step: {len(names) - start}, device time {tot / 1e6:.2f} ms (serialised, cold)")
print()
print("| kernel | launches | total ms | share |")
print("|---|---:|---:|---:|")
for n, (c, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {n} | {c} | {s / 1e6:.3f} | {s / tot * 100:.1f}% |")
