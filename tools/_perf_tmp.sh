cd "${GRAFT_REPO_ROOT:-.}"
for P in 33 49 65 81 97; do
  echo "t=1 P=$P"; python tools/prof_sweep.py --reps 10 --t 1 --nseg $P 2>&1 | tail -1
done
