python tools/prof_sweep.py --reps 20; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_gsrc1.so python tools/prof_sweep.py --reps 20; python tools/prof_sweep.py --reps 20
HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_prof.so python tools/prof_sweep.py --reps 3 2>&1 | grep "pre-action\|separator stage per\|phases"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
