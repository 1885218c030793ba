set -u
# usage: tools/run_ab.sh lib...   (score-phase A/B at 1M, then perf_probe small/big of each library)
for lib in "$@"; do
  FKDE_B200_LIB=$lib timeout 300 python tools/score_ab.py $(basename $lib) 2>&1 | tail -1
done
for lib in "$@"; do
  echo "== $lib"
  FKDE_B200_LIB=$lib timeout 300 python tools/perf_probe.py small big 2>&1 | tail -6
done
