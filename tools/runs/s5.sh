for v in old pf1 pf0 pf2 pf2la1; do
  echo "== $v"
  HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --reps 10 2>&1 | grep -v "Warn\|nan\|^  st\|^  ret\|^  print\|^  f\""
done > gpurun_out/s5.txt 2>&1
cat gpurun_out/s5.txt
