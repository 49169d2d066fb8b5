#!/bin/bash
# Build whole-library ablation variants with extra defines on every source
# (paper_2408_11929_b200/libhelmsweep_<name>.so; load with HELM_LIB=...).
# Usage: tools/abl_lib.sh NAME:DEFINES ...   e.g. tile256:-DHELM_ORTH_TILE=256
set -e
cd "$(dirname "$0")/.."
C=paper_2408_11929_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for spec in "$@"; do
  n=${spec%%:*}; d=${spec#*:}; d=${d//,/ }
  mkdir -p /tmp/abl_$n
  for s in assemble strip_setup sweep_apply sweep_fast sweep_dual krylov; do
    nvcc -c $C/$s.cu -o /tmp/abl_$n/$s.o $F $d &
  done
  wait
  nvcc -shared -o paper_2408_11929_b200/libhelmsweep_$n.so /tmp/abl_$n/*.o -gencode arch=compute_100a,code=sm_100a -lcudart
  echo built $n
done
