HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_prof.so python tools/prof_sweep.py --config 4 --t 1 --reps 3 2>&1 | grep -v "Warn\|^  st\|^  ret\|^  print\|^  f\""
ncu --set full --import-source on --clock-control none -k regex:k_sweep_apply -s 2 -c 1 -o gpurun_out/s44_c4 python tools/prof_sweep.py --config 4 --t 1 --reps 1 --warm 2 > /dev/null 2>&1
