#!/bin/bash
# Quick GPU round trip: K2T parity subset + k2 micro-bench + one bench line.
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tc_ or division or bucket_similarity_random or large_counts or partition" > gpurun_out/quick_tests.log 2>&1
echo "tests_rc=$?"; tail -3 gpurun_out/quick_tests.log
timeout 300 python tools/k2_bench.py > gpurun_out/quick_k2.log 2>&1; echo "k2_rc=$?"; tail -3 gpurun_out/quick_k2.log
timeout 400 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/quick_bench.log 2>&1; echo "bench_rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/quick_bench.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print({k:d[k] for k in ['value','ms_per_step','partition_ms','s5_ms']}, d['phases_ms_rank0'], {k:d['roofline'][k] for k in ['achieved','frac']}, d['e2e']['ms_per_step'] if d.get('e2e') else None)
else:
    print(open('gpurun_out/quick_bench.log').read()[-3000:])
PY
