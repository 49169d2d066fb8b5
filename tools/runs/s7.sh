for v in base nf bp; do echo "== $v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --reps 20 2>&1; done > gpurun_out/s7.txt 2>&1
echo "== both"; python tools/prof_sweep.py --reps 20 >> gpurun_out/s7.txt 2>&1
for v in pbase prof; do echo "== $v"; HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --reps 10 2>&1 | grep -v "Warn\|nan\|^  st\|^  ret\|^  print\|^  f\"\|sub-phases"; done >> gpurun_out/s7.txt 2>&1
cat gpurun_out/s7.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
