for i in 1 2; do
echo "== aa1f410"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_at_aa1f410.so python tools/prof_sweep.py --reps 30
echo "== now"; python tools/prof_sweep.py --reps 30
done
