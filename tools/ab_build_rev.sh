#!/bin/bash
# Build libfkde_b200.so from the sources of git revision REV into ab/lib_NAME.so
# (A/B timing against the working tree):  tools/ab_build_rev.sh HEAD base [-DX=1 ...]
set -eu
cd "$(dirname "$0")/.."
REV=$1; NAME=$2; shift 2
T=$(mktemp -d)
git archive "$REV" paper_2602_10378_b200/csrc include | tar -x -C "$T"
mkdir -p ab
JSON=$(python -c "from paper_2602_10378_b200 import build as B; print(B.json_include())")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC,-O3 -shared "$@" -I "$JSON" -o ab/lib_$NAME.so \
    $(ls "$T"/paper_2602_10378_b200/csrc/*.cu "$T"/paper_2602_10378_b200/csrc/*.cpp) -ldl
rm -rf "$T"
echo ab/lib_$NAME.so
