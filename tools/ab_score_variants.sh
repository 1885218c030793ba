set -u
for v in "default" "noB2:FKDE_NO_B2=1" "noB2_flush1:FKDE_NO_B2=1:flush=1" "sorted_noskip:spatial=3" "dense:spatial=2"; do
  IFS=: read -r label a b <<< "$v"
  envs=""; args=""
  for x in ${a:-} ${b:-}; do case $x in FKDE_*) envs="$envs $x";; *) args="$args $x";; esac; done
  env $envs timeout 300 python tools/score_ab.py $label $args 2>&1 | tail -1
done
