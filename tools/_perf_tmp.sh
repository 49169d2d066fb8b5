cd "${GRAFT_REPO_ROOT:-.}"
for rep in 1 2; do
for v in "" sn0 sn3; do
  if [ -n "$v" ]; then export HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so; else unset HELM_LIB; fi
  echo "== variant ${v:-base}"
  python tools/prof_sweep.py --reps 20 --t 4 2>&1 | tail -1
done
done
