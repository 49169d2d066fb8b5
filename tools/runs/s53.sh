HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_prof.so python tools/prof_sweep.py --reps 3 2>&1 | grep "pre-action\|separator stage per\|phases"
