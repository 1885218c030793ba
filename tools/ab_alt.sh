#!/bin/bash
# Interleaved A/B of library variants on the bench workload (runs on the GPU box):
#   tools/ab_alt.sh ROUNDS lib_a lib_b ...   (names under ab/ without .so)
# one perf_probe bench1m per (round, variant), variants alternating, so clock /
# power drift hits every variant alike
cd "$(dirname "$0")/.."
R=$1; shift
for i in $(seq 1 "$R"); do
  for L in "$@"; do
    echo -n "$L "; FKDE_B200_LIB=ab/$L.so timeout 120 python tools/perf_probe.py bench1m 2>&1 | tail -1
  done
done
