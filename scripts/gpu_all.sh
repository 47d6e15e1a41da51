#!/bin/bash
# All GPU tests (stop at first failure) + one bench line (no e2e).
cd "$(dirname "$0")/.."
L=${1:-r02k}
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/${L}_tests.log 2>&1; echo "tests_rc=$?"; tail -25 gpurun_out/${L}_tests.log | grep -v "Warn\|warn\|fork" | tail -15
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/${L}_bench.log 2>&1; echo "bench_rc=$?"
python - <<PY
import json
l=[x for x in open('gpurun_out/${L}_bench.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print({k:d[k] for k in ['value','ms_per_step','partition_ms','s5_ms']}); print({k:round(v,3) for k,v in d['phases_ms_rank0'].items()}); print({k:d['roofline'][k] for k in ['bound','frac','frac_tensor_method','frac_hbm','kernel_ms']})
else:
    print(open('gpurun_out/${L}_bench.log').read()[-3000:])
PY
