cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in "" _rot0 _m4 _m4u1 _m4r0; do echo "== lib$v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep$v.so REPS=4 python tools/prof_setup.py 5 2>&1 | tail -1; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep$v.so PAR_SETUP=1 REPS=4 python tools/prof_setup.py 5 2>&1 | tail -1; done > $O/s57_setup.txt 2>&1
cat $O/s57_setup.txt
