python tools/prof_sweep.py --reps 20
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
