ncu --set full --import-source on --clock-control none -k regex:k_sweep_dual -s 2 -c 1 -o gpurun_out/s28_two python tools/prof_sweep.py --reps 1 --warm 2 > gpurun_out/s28_ncu.log 2>&1
cat > /tmp/full.py <<'PY'
import runpy, sys
import paper_2408_11929_b200 as hs
hs.set_knob("sep_full", 1)
sys.argv = ["prof_sweep.py", "--reps", "1", "--warm", "2"]
runpy.run_path("tools/prof_sweep.py", run_name="__main__")
PY
PYTHONPATH=$PWD ncu --set full --import-source on --clock-control none -k regex:k_sweep_dual -s 2 -c 1 -o gpurun_out/s28_full python /tmp/full.py >> gpurun_out/s28_ncu.log 2>&1
ls -la gpurun_out/s28*
