#!/bin/bash
# bench.py on every BASELINE config (runs on the GPU box): gpurun_out/bench_w{K}.json
# and one summary line per config on stdout
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in ${WORKLOADS:-1 2 3 4 5}; do
    steps=200; [ "$w" = 5 ] && steps=5; [ "$w" = 4 ] && steps=50
    timeout 300 python bench.py --workload $w --steps $steps --warmup 5 ${BENCH_ARGS:-} \
        > gpurun_out/bench_w$w.json 2> gpurun_out/bench_w$w.err || { echo "w$w failed"; tail -3 gpurun_out/bench_w$w.err; continue; }
    python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
d = json.load(open(f"gpurun_out/bench_w{w}.json"))
sk = d["roofline"]["tile_skipping"]
print(f"w{w} ms/step {d['ms_per_step']:.4f} value {d['value']:.4g} e2e {d['e2e']['value']:.4g} "
      f"phases {d['phases_ms']} frac {d['roofline']['frac']:.3f} launches/step "
      f"{d['gpu_launches'] / d['steps']:.0f} sm_mhz {d['clocks']['sm_mhz']} "
      f"skipped {sk['tiles_skipped']}/{sk['tiles_total']} d {sk['density']['tiles_skipped']}/{sk['density']['tiles_total']}")
PY
done
