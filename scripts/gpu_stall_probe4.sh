#!/bin/bash
# Config 3's tenth-step outlier: does a stream-ordered pool allocation hold the host? (SA_TRACE_ALLOC=1)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
SA_TRACE_ALLOC=1 python bench.py --config 3 --steps 12 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/stall4_$r.log 2> gpurun_out/stall4_$r.err
grep -c "held the host" gpurun_out/stall4_$r.err; grep "held the host" gpurun_out/stall4_$r.err | tail -8
python -c "
import json
l=[x for x in open('gpurun_out/stall4_$r.log') if x.startswith('{')]
d=json.loads(l[-1]); print('step', d['step_ms_rank0']); print('S2a', d['phase_steps_ms_rank0']['S2a'])
"
done
