#!/bin/bash
# Density-pass skip threshold (FKDE_DENSITY_SKIP, half r^2 in log2 units proven by the
# tile boxes; default kDensitySkipHalfR2) on the bench workload: phase times, skipped
# density tiles and rows sent to the direct recompute, interleaved
cd "$(dirname "$0")/.."
for v in ${VALUES:-45 43 41.5 45 43 41.5}; do
  echo -n "skip=$v "; FKDE_DENSITY_SKIP=$v WORKLOADS=5 BENCH_ARGS="--no-cpu-baseline --steps 3" bash tools/bench_all.sh | cut -c1-330
  python -c "import json;d=json.load(open('gpurun_out/bench_w5.json'));print('   ', json.dumps(d['roofline']['tile_skipping']))"
done
