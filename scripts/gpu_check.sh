#!/bin/bash
# Full GPU test suite + one short phase bench (default configuration).
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/check_tests.log 2>&1; echo "tests_rc=$?"; tail -3 gpurun_out/check_tests.log
python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bp.log 2>&1 || tail -5 gpurun_out/bp.log
python - <<'PY'
import json
d = json.loads([x for x in open('gpurun_out/bp.log') if x.startswith('{')][-1])
ph = d['phases_ms_rank0']; r = d['roofline']
print(f"step {d['ms_per_step']:.2f} S2a {ph['S2a']:.2f} S2d {ph['S2d']:.2f} S5 {ph['S5']:.2f} gemm {ph['S5_gemm']:.2f} "
      f"frac {r['frac']:.3f} phase_frac {r['phase_frac']:.3f} {r['operand']} {d['dtype']}")
PY
