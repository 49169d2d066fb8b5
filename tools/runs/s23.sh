for n in 33 36 37 36 37; do python tools/prof_sweep.py --reps 30 --nseg $n; done
