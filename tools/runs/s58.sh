cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in "" _xs0 "" _xs0; do echo "== lib$v"; for t in 4 2 1; do HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep$v.so python tools/prof_sweep.py --t $t --reps 20 2>&1 | tail -1; done; done > $O/s58_sweep.txt 2>&1
cat $O/s58_sweep.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/s58_pytest.log 2>&1; tail -3 $O/s58_pytest.log
