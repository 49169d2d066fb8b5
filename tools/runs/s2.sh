for n in 33 35 36 37; do python tools/prof_sweep.py --reps 20 --nseg $n; done > gpurun_out/s2_nseg.txt 2>&1
HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_prof.so python tools/prof_sweep.py --reps 3 --nseg 37 >> gpurun_out/s2_nseg.txt 2>&1
cat gpurun_out/s2_nseg.txt | grep -v Warn
