set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/prof_sweep.py --reps 20 > gpurun_out/s1_prof.txt 2>&1
HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_prof.so python tools/prof_sweep.py --reps 5 >> gpurun_out/s1_prof.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s1_pytest.txt 2>&1
tail -3 gpurun_out/s1_pytest.txt
python bench.py > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err
tail -c 3000 gpurun_out/s1_bench.json
