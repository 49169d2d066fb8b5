cd "${GRAFT_REPO_ROOT:-.}"
for rep in 1 2; do
for v in "" gsrc0; do
  if [ -n "$v" ]; then export HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so; else unset HELM_LIB; fi
  echo "== variant ${v:-base}"
  python tools/prof_sweep.py --reps 20 --t 4 2>&1 | tail -1
done
done
unset HELM_LIB
python -m pytest tests/test_gpu_parity.py -x -q -k "sweep_apply_parity or kernels_parity or short_segments or tiny or single_sweep" 2>&1 | tail -2
