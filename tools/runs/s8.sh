ncu --set full --import-source on --clock-control none -k regex:k_sweep_dual -s 2 -c 1 -o gpurun_out/s8_dual python tools/prof_sweep.py --reps 1 --warm 2 > gpurun_out/s8_ncu.log 2>&1
ls -la gpurun_out/
