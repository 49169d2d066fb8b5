for v in e4 e8 e16; do echo "== $v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --reps 20 2>&1; done > gpurun_out/s9.txt 2>&1
echo "== default" >> gpurun_out/s9.txt; python tools/prof_sweep.py --reps 20 >> gpurun_out/s9.txt 2>&1
for n in 34 35 36; do echo "== nseg $n"; python tools/prof_sweep.py --reps 20 --nseg $n; done >> gpurun_out/s9.txt 2>&1
cat gpurun_out/s9.txt
