for n in 41 49 57 65 73; do python tools/prof_sweep.py --t 1 --reps 20 --nseg $n; done
for n in 36 41 49 57 65 73; do python tools/prof_sweep.py --t 2 --reps 20 --nseg $n; done
