#!/bin/bash
# S5 GEMM component times via SA_K2T_DEBUG switches (1 no MMA, 2 no TMA loads, 4 no epilogue, 8 no matrix stores, 64 F without fp64).
cd "$(dirname "$0")/.."
L=${1:-r02o}
for d in ${DBGS:-0 8 64 72 4 5}; do
  SA_K2T_DEBUG=$d timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 2 > gpurun_out/${L}_d$d.log 2>&1
  python - <<PY
import json
l=[x for x in open('gpurun_out/${L}_d$d.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('dbg $d', d and round(d['ms_per_step'],3), d and {k: round(v,3) for k,v in d['phases_ms_rank0'].items() if k in ('S5_gemm','S2a_gemm','S2d_gemm')})
PY
done
