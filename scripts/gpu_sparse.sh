#!/bin/bash
# Sparse-layer parity tests, then the K2T parity subset, then one bench line.
cd "$(dirname "$0")/.."
L=${1:-r02b}
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q > gpurun_out/${L}_sparse.log 2>&1; echo "sparse_rc=$?"; tail -30 gpurun_out/${L}_sparse.log | grep -v Warning | tail -25
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${L}_parity.log 2>&1; echo "parity_rc=$?"; tail -3 gpurun_out/${L}_parity.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/${L}_bench.log 2>&1; echo "bench_rc=$?"
python - <<PY
import json
l=[x for x in open('gpurun_out/${L}_bench.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print({k:d[k] for k in ['value','ms_per_step','partition_ms','s5_ms']}); print(d['phases_ms_rank0']); print({k:d['roofline'][k] for k in ['bound','frac','frac_tensor_method','frac_hbm','kernel_ms','kprime']})
else:
    print(open('gpurun_out/${L}_bench.log').read()[-3000:])
PY
