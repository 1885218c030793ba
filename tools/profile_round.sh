#!/bin/bash
# Runs on the GPU box (under gpurun).  Produces, in gpurun_out/:
#   launches.csv            every kernel launch of a short bench run with its device time
#   prof_1m.ncu-rep         ncu --set full of the score-pass kernel at the headline size
#                           (n = 2^20, m = 2^17)
#   prof_1m_q.ncu-rep       the density-pass kernel of the same run
#   prof_32k.ncu-rep        score + density kernels at n = m = 32768
# then: python tools/summarize_ncu.py gpurun_out/prof_1m.ncu-rep gpurun_out/prof_1m_q.ncu-rep \
#         gpurun_out/prof_32k.ncu-rep --launches gpurun_out/launches.csv --out profiles/<round>
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/launches_bench.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:pairwise_tc_kernel -s 0 -c 1 -o gpurun_out/prof_1m -f \
    python tools/perf_probe.py sd1m > gpurun_out/prof_1m.log 2>&1
echo "ncu 1m score rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:pairwise_tc_kernel -s 1 -c 1 -o gpurun_out/prof_1m_q -f \
    python tools/perf_probe.py sd1m > gpurun_out/prof_1m_q.log 2>&1
echo "ncu 1m density rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:pairwise_tc_kernel -s 2 -c 2 -o gpurun_out/prof_32k -f \
    python tools/perf_probe.py sd32k > gpurun_out/prof_32k.log 2>&1
echo "ncu 32k rc=$?"
