#!/bin/bash
# flush_sweep (accuracy + n=262144 score-pass time) for each ab/ variant
cd "$(dirname "$0")/.."
F=${FLUSH:-2}
for L in "$@"; do
  FKDE_B200_LIB=ab/$L.so timeout 180 python tools/flush_sweep.py $F 2>&1 | grep flush=
done
