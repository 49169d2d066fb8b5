cd $GRAFT_REPO_ROOT
O=gpurun_out
for U in 1 3 9; do ./tools/bench_gj_u$U 2>&1 | grep -A1 "rotating\|row_invert (LPR" ; done > $O/s56_gj.txt
for v in "" _rot0 _up1 _up2; do echo "== lib$v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep$v.so REPS=4 python tools/prof_setup.py 5 2>&1 | tail -2; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep$v.so PAR_SETUP=1 REPS=4 python tools/prof_setup.py 5 2>&1 | tail -2; done > $O/s56_setup.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or fullsize or fd5" > $O/s56_pytest.log 2>&1; tail -2 $O/s56_pytest.log
cat $O/s56_gj.txt $O/s56_setup.txt
