for v in sx1p sx2p; do echo "== $v"; HELM_SKEW=1 HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --reps 3 2>&1 | grep -v "Warn\|nan\|^  st\|^  ret\|^  print\|^  f\"\|sub-phases" | head -10; done
for v in sx1 sx2; do echo "== $v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --reps 20; done
echo "== default"; python tools/prof_sweep.py --reps 20
