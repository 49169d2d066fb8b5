#!/bin/bash
# End-of-round evidence for profiles/ (run on the B200 box via gpurun):
#   tools/profile_round.sh TAG   -> gpurun_out/TAG_*
# bench line, reference arm, per-kernel launch list of one bench step, ncu
# --set full captures of the sweep / orthogonalisation / factorisation kernels,
# and the per-config report table.  Each ncu command runs only after the same
# command has exited 0 without ncu (bench.py / prof_sweep.py / prof_setup.py).
set -x
T=${1:-rXX}
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out
timeout 300 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err || exit 1
timeout 300 python bench.py --impl reference > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err
timeout 120 python tools/prof_sweep.py --reps 1 > /dev/null 2>&1 || exit 1
timeout 120 python tools/prof_setup.py 5 > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep_dual -s 2 -c 1 -o $O/${T}_dual \
  python tools/prof_sweep.py --reps 1 > $O/${T}_ncu_dual.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_orth -s 11 -c 1 -o $O/${T}_orth \
  python tools/prof_setup.py 5 > $O/${T}_ncu_orth.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_factor_rows|k_reduced" -s 0 -c 3 -o $O/${T}_setup \
  python tools/prof_setup.py 5 > $O/${T}_ncu_setup.log 2>&1
timeout 1500 python tools/report.py > $O/${T}_report.md 2> $O/${T}_report.err
ls -la $O
