#!/bin/bash
# One bench.py line per BASELINE config (configs[0-3]; configs[4] is the
# default bench), written to gpurun_out/bench_<config>.json.
#   bash scripts/bench_configs.sh [steps]
set -u
mkdir -p gpurun_out
for cfg in tiny block layered hetero; do
  steps=${1:-}
  if [ -z "$steps" ]; then
    case $cfg in tiny|block) steps=20;; layered) steps=5;; *) steps=2;; esac
  fi
  timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?"
done
