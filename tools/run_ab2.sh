set -u
for lib in "$@"; do
  FKDE_B200_LIB=$lib timeout 300 python tools/score_ab.py $(basename $lib) 2>&1 | tail -1
done
