#!/bin/bash
# A/B timing + accuracy of library variants under ab/ (run on the GPU box).
#   tools/ab_run.sh lib_a lib_b ...   (names without ab/ and .so)
cd "$(dirname "$0")/.."
for L in "$@"; do
  FKDE_B200_LIB=ab/$L.so timeout 180 python tools/flush_sweep.py 2 2>&1 | tail -1
  FKDE_B200_LIB=ab/$L.so timeout 180 python tools/perf_probe.py sd1m 2>&1 | tail -1
done
