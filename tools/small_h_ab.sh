#!/bin/bash
# small_h_probe.py on library variants under ab/, interleaved: tools/small_h_ab.sh R lib_a lib_b ...
cd "$(dirname "$0")/.."
R=$1; shift
for i in $(seq 1 "$R"); do for L in "$@"; do echo "== $L"; FKDE_B200_LIB=ab/$L.so python tools/small_h_probe.py | grep "h0/3"; done; done
