#!/bin/bash
# Repeated short bench runs: per-step device times and host enqueue segments (outlier hunt).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in $(seq ${RUNS:-6}); do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/outl_$i.log 2>&1
  python - gpurun_out/outl_$i.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l)
st=d['step_ms_rank0']; hs=d['host_segments_ms_rank0']
bad=[i for i,x in enumerate(st) if x>12]
print('ms/step %.3f steps %s' % (d['ms_per_step'], st))
for i in bad: print('  outlier step', i, 'host segments', hs[i])
print('  host seg medians', [round(sorted(h[j] for h in hs)[len(hs)//2],2) for j in range(len(hs[0]))])
PY
done
