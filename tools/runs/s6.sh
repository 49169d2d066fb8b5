for v in o0x0 o1x0 o1x1 o1x1pf2; do
  echo "== $v"
  HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --reps 10 2>&1 | grep -v "Warn\|nan\|^  st\|^  ret\|^  print\|^  f\"\|sub-phases"
done > gpurun_out/s6.txt 2>&1
for v in n_o1x0 n_o1x1; do echo "== $v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --reps 20 2>&1; done >> gpurun_out/s6.txt 2>&1
cat gpurun_out/s6.txt
