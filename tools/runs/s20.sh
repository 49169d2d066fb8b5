for v in xb1 xb1la1; do echo "== $v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --reps 20; done
echo "== default"; python tools/prof_sweep.py --reps 20
HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_xb1p.so python tools/prof_sweep.py --reps 3 2>&1 | grep -v "Warn\|nan\|^  st\|^  ret\|^  print\|^  f\"\|sub-phases" | head -10
