for v in default noxc; do
  L=$PWD/paper_2408_11929_b200/libhelmsweep.so; [ $v = noxc ] && L=$PWD/paper_2408_11929_b200/libhelmsweep_noxc.so
  echo "== $v"; HELM_LIB=$L REPS=3 python tools/prof_setup.py 5 2>&1 | tail -2
  HELM_LIB=$L REPS=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_factor|k_reduced|k_strip" --csv python tools/prof_setup.py 5 2>/dev/null | grep -v "^==" | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
from collections import defaultdict
d=defaultdict(list)
for r in rows[1:]:
  if len(r)>vi: d[r[ki][:40]].append(float(r[vi].replace(',','')))
for k,v in d.items(): print(f'  {k:40s} n={len(v)} mean={sum(v)/len(v)/1e6:.3f} ms')
"
done > gpurun_out/s10.txt 2>&1
cat gpurun_out/s10.txt
