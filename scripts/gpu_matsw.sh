#!/bin/bash
# S5 epilogue variants: matrix-epilogue warps 16 / 8, TMA stores on / off.
cd "$(dirname "$0")/.."
L=${1:-r02n}
for cfg in "16 1" "8 1" "16 0"; do
  set -- $cfg
  SA_K2T_MATSW=$1 SA_K2T_TMA_STORE=$2 timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${L}_m$1_t$2.log 2>&1
  python - <<PY
import json
l=[x for x in open('gpurun_out/${L}_m$1_t$2.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('matsw $1 tma $2', d and round(d['ms_per_step'],3), d and {k: round(v,3) for k,v in d['phases_ms_rank0'].items() if k in ('S5','S5_gemm','S2a_gemm')})
PY
done
