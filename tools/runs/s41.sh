cat > /tmp/two.py <<'PY'
import runpy, sys
import paper_2408_11929_b200 as hs
hs.set_knob("sep_two_level", 1)
sys.argv = ["prof_sweep.py"] + sys.argv[1:]
runpy.run_path("tools/prof_sweep.py", run_name="__main__")
PY
for n in 49 65 73 81; do PYTHONPATH=$PWD python /tmp/two.py --t 1 --reps 20 --nseg $n; done
for n in 41 57 73; do PYTHONPATH=$PWD python /tmp/two.py --t 2 --reps 20 --nseg $n; done
for n in 36; do PYTHONPATH=$PWD python /tmp/two.py --t 4 --reps 20 --nseg $n; done
