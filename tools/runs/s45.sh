for v in gxpf0 gxpipe; do echo "== $v"; for t in 1 4; do HELM_LIB=$PWD/paper_2408_11929_b200/libhelmsweep_$v.so python tools/prof_sweep.py --config 4 --t $t --reps 5; done; done
echo "== default"; for t in 1 4; do python tools/prof_sweep.py --config 4 --t $t --reps 5; done
