python tools/prof_sweep.py --reps 20 > gpurun_out/s4.txt 2>&1
for n in 36 37; do python tools/prof_sweep.py --reps 20 --nseg $n; done >> gpurun_out/s4.txt 2>&1
HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_prof.so python tools/prof_sweep.py --reps 3 >> gpurun_out/s4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q >> gpurun_out/s4.txt 2>&1
grep -v Warn gpurun_out/s4.txt | grep -v "^  print\|^  f\"\|nan"
