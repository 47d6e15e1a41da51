#!/bin/bash
# Config 3's tenth-step outlier: device time per step segment and per libsa phase.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
python bench.py --config 3 --steps 12 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/stall2_$r.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/stall2_$r.log') if x.startswith('{')]
d=json.loads(l[-1])
print('step', d['step_ms_rank0']); print('devseg', d['device_segments_ms_rank0'][7:11]); print('hostseg', d['host_segments_ms_rank0'][7:11])
for k,v in d['phase_steps_ms_rank0'].items(): print(k, v)
"
done
