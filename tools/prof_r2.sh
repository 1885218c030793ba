set -u
mkdir -p gpurun_out
FKDE_B200_LIB=ab/lib_cta.so timeout 300 python tools/cta_balance.py > gpurun_out/cta_balance.log 2>&1; echo "cta rc=$?"; cat gpurun_out/cta_balance.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/launches_bench.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:pairwise_tc_kernel -s 1 -c 1 -o gpurun_out/prof_1m_score -f \
    python tools/perf_probe.py sd1m > gpurun_out/prof_1m.log 2>&1; echo "ncu score rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:pairwise_tc_kernel -s 0 -c 1 -o gpurun_out/prof_1m_check -f \
    python tools/perf_probe.py sd1m > gpurun_out/prof_1m_c.log 2>&1; echo "ncu check rc=$?"
