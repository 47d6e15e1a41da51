#!/bin/bash
# S5 epilogue A/B: TMA tensor stores vs per-thread stores; ncu of the S5 GEMM.
cd "$(dirname "$0")/.."
L=${1:-r02l}
for t in 1 0; do
  SA_K2T_TMA_STORE=$t timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${L}_tma$t.log 2>&1
  python - <<PY
import json
l=[x for x in open('gpurun_out/${L}_tma$t.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('tma $t', d and round(d['ms_per_step'],3), d and {k: round(v,3) for k,v in d['phases_ms_rank0'].items() if k in ('S5','S5_gemm','S2a_gemm')})
PY
done
KREGEX="regex:gemm2_kernel<sa::KeyMatEpi<6>" COUNT=1 bash scripts/gpu_ncu_kernels.sh ${L}
