#!/bin/bash
# End-of-round evidence for profiles/ (run on the B200 box via gpurun):
#   tools/profile_round.sh TAG   -> gpurun_out/TAG_*
# bench line, reference arm, per-kernel launch list of one bench step, ncu
# --set full captures of the sweep / SpMM / orthogonalisation / factorisation
# kernels, and the per-config report table.  Each ncu command runs only after
# the same command has exited 0 without ncu.
set -x
T=${1:-rXX}
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err || exit 1
timeout 600 python bench.py --impl reference > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err
timeout 120 python tools/prof_sweep.py --reps 1 > $O/${T}_prof_sweep.txt 2>&1 || exit 1
timeout 120 python tools/prof_spmm.py 2 > $O/${T}_prof_spmm.txt 2>&1 || exit 1
timeout 120 python tools/prof_setup.py 5 > $O/${T}_prof_setup.txt 2>&1 || exit 1
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-north-star > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-north-star > $O/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep_dual -s 2 -c 1 -o $O/${T}_dual \
  python tools/prof_sweep.py --reps 1 > $O/${T}_ncu_dual.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm -s 1 -c 4 -o $O/${T}_spmm \
  python tools/prof_spmm.py 2 > $O/${T}_ncu_spmm.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_orth -s 11 -c 1 -o $O/${T}_orth \
  python tools/prof_setup.py 5 > $O/${T}_ncu_orth.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_factor_rows|k_reduced" -s 0 -c 3 -o $O/${T}_setup \
  python tools/prof_setup.py 5 > $O/${T}_ncu_setup.log 2>&1
timeout 1500 python tools/report.py > $O/${T}_report.md 2> $O/${T}_report.err
ls -la $O
