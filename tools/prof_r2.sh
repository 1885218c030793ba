#!/bin/bash
# Round-2 profile capture (runs on the GPU box under gpurun), into gpurun_out/:
#   launches_r2.csv   every kernel launch of a short bench run (gpu__time_duration)
#   prof_1m_score / prof_1m_check / prof_1m_density .ncu-rep: ncu --set full of the
#   score, check and density kernels on the bench workload (perf_probe bench1m)
# then: python tools/summarize_ncu.py gpurun_out/prof_1m_score.ncu-rep ... --launches gpurun_out/launches_r2.csv --out profiles/round2
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/launches_bench.log 2>&1; echo "launch list rc=$?"
# bench1m runs the SD-KDE twice (warm-up + timed): kernel order per call is
# check (<3>), score (<0>), density (<1>)
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:pairwise_tc_kernel -s 4 -c 1 -o gpurun_out/prof_1m_score -f \
    python tools/perf_probe.py bench1m > gpurun_out/prof_1m.log 2>&1; echo "ncu score rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:pairwise_tc_kernel -s 3 -c 1 -o gpurun_out/prof_1m_check -f \
    python tools/perf_probe.py bench1m > gpurun_out/prof_1m_c.log 2>&1; echo "ncu check rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:pairwise_tc_kernel -s 5 -c 1 -o gpurun_out/prof_1m_density -f \
    python tools/perf_probe.py bench1m > gpurun_out/prof_1m_d.log 2>&1; echo "ncu density rc=$?"
