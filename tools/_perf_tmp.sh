cd "${GRAFT_REPO_ROOT:-.}"
for v in "" nos nowops novin noxmv; do
  if [ -n "$v" ]; then export HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so; else unset HELM_LIB; fi
  echo "== variant ${v:-base}"
  python tools/prof_sweep.py --reps 10 --t 4 2>&1 | tail -1
done
for v in prof profstep; do
  export HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so; export HELM_CYCLES=1
  echo "== variant $v"
  python tools/prof_sweep.py --reps 3 --t 4 2>&1 | tail -6
  python tools/prof_sweep.py --reps 3 --t 1 2>&1 | tail -6
done
