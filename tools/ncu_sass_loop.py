"""Print the SASS of the hottest loop body (instructions sharing the most
common high execution count) from `ncu -i X --page source --csv --print-source sass`,
with per-instruction stall samples and the top stall reasons."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
body = []
for r in rows[2:]:
    try:
        body.append((int(r[ie]), int(r[ws]), r))
    except ValueError:
        pass
cnt = collections.Counter(n for n, _, _ in body)
want = int(sys.argv[2]) if len(sys.argv) > 2 else max(cnt, key=lambda n: n * cnt[n] if n > 1000 else 0)
sel = [b for b in body if b[0] == want]
tot = sum(s for _, s, _ in sel) or 1
print(f"count {want}: {len(sel)} instructions, {tot} samples")
agg = collections.Counter()
for n, s, r in sel:
    reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in st), reverse=True)[:3]
    for v, k in reasons:
        agg[k] += v
    rs = " ".join(f"{k}:{v}" for v, k in reasons if v)
    print(f"{s:6d} {r[1].strip()[:70]:70s} {rs}")
print(agg.most_common(8))
