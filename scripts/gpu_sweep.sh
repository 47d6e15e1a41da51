#!/bin/bash
# Phase-bench sweep over env knobs: scripts/gpu_sweep.sh "LABEL:ENV=.. ENV=.." ...
cd "$(dirname "$0")/.."
for spec in "$@"; do
  label=${spec%%:*}; envs=${spec#*:}
  env $envs bash scripts/bench_phases.sh "$label" 2>&1 | tail -1
done
