#!/bin/bash
# Bench lines for each key-epilogue warp count (S2a / S2d GEMMs).
cd "$(dirname "$0")/.."
L=${1:-r02d}
for w in 8 12 16; do
  SA_K2T_KEYSW=$w timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${L}_keysw$w.log 2>&1
  python - <<PY
import json
l=[x for x in open('gpurun_out/${L}_keysw$w.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('keysw $w', d and round(d['ms_per_step'],3), d and {k: round(v,3) for k,v in d['phases_ms_rank0'].items()})
PY
done
