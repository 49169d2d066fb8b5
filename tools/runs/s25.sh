timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_level" 2>&1 | tail -15
python tools/prof_sweep.py --reps 20
HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_prof.so python tools/prof_sweep.py --reps 3 2>&1 | grep "separator stage per\|phases\|pre-actions ("
