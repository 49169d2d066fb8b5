M="dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum"
for v in l2p4 l2p2; do echo "== $v"; HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --reps 20
HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so ncu --metrics $M --clock-control none -k regex:k_sweep_dual -s 2 -c 1 python tools/prof_sweep.py --reps 1 --warm 2 2>&1 | grep -E "dram__bytes|hit_rate|duration|persist"; done
echo "== default"; python tools/prof_sweep.py --reps 20
