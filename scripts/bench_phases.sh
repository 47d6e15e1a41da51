#!/bin/bash
# One short bench run, phases only: scripts/bench_phases.sh [label]
cd "$(dirname "$0")/.."
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bp.log 2>&1 || { tail -5 gpurun_out/bp.log; exit 1; }
python - "$1" <<'PY'
import json, sys
d = json.loads([x for x in open('gpurun_out/bp.log') if x.startswith('{')][-1])
ph = d['phases_ms_rank0']
print(sys.argv[1], f"step {d['ms_per_step']:.2f}  S2a {ph['S2a']:.2f}  S2d {ph['S2d']:.2f}  S5 {ph['S5']:.2f}  frac {d['roofline']['frac']:.3f}")
PY
