#!/bin/bash
# Per-config measurements (runs on the GPU box under gpurun), into gpurun_out/:
#   bench_w{1..5}.json   bench.py --workload K (K = BASELINE.json config number)
#   launches_w{K}.csv    every kernel launch of a short bench run (gpu__time_duration)
#   prof_w{K}.ncu-rep    ncu --set full of the dominant kernel (config 2: the score
#                        kernel of the second step; configs 3/4: the density kernel)
# then: python tools/summarize_ncu.py gpurun_out/prof_w2.ncu-rep ... \
#         --launches-glob 'gpurun_out/launches_w*.csv' --out profiles/round2_configs
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in 1 2 3 4 5; do
    steps=200; [ "$w" = 5 ] && steps=5; [ "$w" = 4 ] && steps=50
    timeout 300 python bench.py --workload $w --steps $steps --warmup 5 > gpurun_out/bench_w$w.json \
        2> gpurun_out/bench_w$w.err; echo "bench w$w rc=$?"
done
for w in 1 2 3 4; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
        --log-file gpurun_out/launches_w$w.csv python bench.py --workload $w --steps 2 --warmup 3 \
        --no-cpu-baseline > /dev/null 2>&1; echo "launches w$w rc=$?"
done
# kernel order per SD-KDE step on the spatial order: check <3>, score <0>, density <1>
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pairwise_tc_kernel \
    -s 4 -c 1 -o gpurun_out/prof_w2 -f python bench.py --workload 2 --steps 1 --warmup 3 \
    --no-cpu-baseline > /dev/null 2>&1; echo "ncu w2 rc=$?"
for w in 3 4; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:pairwise_tc_kernel \
        -s 1 -c 1 -o gpurun_out/prof_w$w -f python bench.py --workload $w --steps 1 --warmup 3 \
        --no-cpu-baseline > /dev/null 2>&1; echo "ncu w$w rc=$?"
done
