#!/bin/bash
# Build ablation variants of k_sweep_dual as whole libraries
# (paper_2408_11929_b200/libhelmsweep_<name>.so; load with HELM_LIB=...).
# Usage: tools/abl_build.sh NAME:DEFINES ...   e.g. novin:-DHELM_DUAL_ABL_NOVIN
set -e
cd "$(dirname "$0")/.."
C=paper_2408_11929_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
mkdir -p /tmp/abl
for s in assemble strip_setup sweep_apply sweep_fast krylov; do
  [ /tmp/abl/$s.o -nt $C/$s.cu ] || nvcc -c $C/$s.cu -o /tmp/abl/$s.o $F &
done
wait
for spec in "$@"; do
  n=${spec%%:*}; d=${spec#*:}; d=${d//,/ }
  nvcc -c $C/sweep_dual.cu -o /tmp/abl/dual_$n.o $F $d
  nvcc -shared -o paper_2408_11929_b200/libhelmsweep_$n.so /tmp/abl/{assemble,strip_setup,sweep_apply,sweep_fast,krylov}.o /tmp/abl/dual_$n.o -gencode arch=compute_100a,code=sm_100a -lcudart
  echo built $n
done
