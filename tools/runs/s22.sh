for n in 33 34 35 36; do python tools/prof_sweep.py --reps 20 --nseg $n; done
for n in 34 36; do HELM_SKEW=1 HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_prof.so python tools/prof_sweep.py --reps 3 --nseg $n 2>&1 | grep "separator stage per\|phases" ; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
