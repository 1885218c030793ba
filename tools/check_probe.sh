#!/bin/bash
# Check-pass trade-off at n = 2^20: SD-KDE with the predictor threshold
# FKDE_SKIP_PRED (centroid half-distance^2 in log2 units above which a tile pair is
# checked; default kSkipPredict) swept, and 1e9 = nothing predicted (only the
# box-proven tiles skipped, no check work) -- tile counts and phase times
cd "$(dirname "$0")/.."
for p in ${PREDS:-"" 1e9}; do
    FKDE_SKIP_PRED=$p WORKLOADS=5 BENCH_ARGS="--no-cpu-baseline --steps 3" bash tools/bench_all.sh | sed "s/^/pred=${p:-default} /"
    python -c "import json;d=json.load(open('gpurun_out/bench_w5.json'));print(json.dumps(d['roofline']['tile_skipping']))"
done
