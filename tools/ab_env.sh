#!/bin/bash
# Same-box A/B of env knobs: tools/ab_env.sh "<dp_ab args>" "VAR=a VAR2=b" "VAR=c" ...
args=$1; shift
for envs in "" "$@"; do
  echo "== [${envs}]"
  env $envs MODES=${MODES:-0} python tools/dp_ab.py $args 2>&1 | grep early_exit=True
done
