cat > /tmp/full.py <<'PY'
import runpy, sys
import paper_2408_11929_b200 as hs
hs.set_knob("sep_full", 1)
sys.argv = ["prof_sweep.py"] + sys.argv[1:]
runpy.run_path("tools/prof_sweep.py", run_name="__main__")
PY
M="dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum"
for v in default nox nox0; do L=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so; [ $v = default ] && L=$PWD/paper_2408_11929_b200/libhelmsweep.so
 echo "== two-level $v"; HELM_LIB=$L ncu --metrics $M --clock-control none -k regex:k_sweep_dual -s 2 -c 1 python tools/prof_sweep.py --reps 1 --warm 2 2>&1 | grep -E "dram__bytes|hit_rate|duration"
 echo "== full $v"; HELM_LIB=$L PYTHONPATH=$PWD ncu --metrics $M --clock-control none -k regex:k_sweep_dual -s 2 -c 1 python /tmp/full.py --reps 1 --warm 2 2>&1 | grep -E "dram__bytes|hit_rate|duration"
done
