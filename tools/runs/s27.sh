echo "== default (XCH 4, two-level)"; python tools/prof_sweep.py --reps 20
echo "== XCH 6 two-level"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_x6.so python tools/prof_sweep.py --reps 20
cat > /tmp/full.py <<'PY'
import runpy, sys
import paper_2408_11929_b200 as hs
hs.set_knob("sep_full", 1)
sys.argv = ["prof_sweep.py", "--reps", "20"]
runpy.run_path("tools/prof_sweep.py", run_name="__main__")
PY
echo "== XCH 4 full"; PYTHONPATH=$PWD python /tmp/full.py
echo "== XCH 6 full"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_x6.so PYTHONPATH=$PWD python /tmp/full.py
HELM_CYCLES=1 HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_x6p.so python tools/prof_sweep.py --reps 3 2>&1 | grep "separator stage per\|phases\|two-level"
