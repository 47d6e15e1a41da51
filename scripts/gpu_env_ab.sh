#!/bin/bash
# A/B of one environment switch on the bench (phases + GEMM times), alternating runs.
# usage: gpu_env_ab.sh LABEL VAR "v1 v2 ..." [reps]
cd "$(dirname "$0")/.."
L=$1; VAR=$2; VALS=$3; REPS=${4:-2}
for r in $(seq 1 $REPS); do for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${L}_$v.log 2>&1
  python - <<PY
import json
l=[x for x in open('gpurun_out/${L}_$v.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$VAR=$v', d and round(d['ms_per_step'],3), d and {k: round(v,3) for k,v in d['phases_ms_rank0'].items() if k in ('S2a','S2d','S5','S5_gemm','S2a_gemm','S2d_gemm')})
PY
done; done
