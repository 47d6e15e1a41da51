#!/bin/bash
# Tests (sparse + parity), then the ncu launch list of one bench step (per-kernel time shares).
cd "$(dirname "$0")/.."
L=${1:-r02c}
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q > gpurun_out/${L}_sparse.log 2>&1; echo "sparse_rc=$?"; tail -30 gpurun_out/${L}_sparse.log | grep -v Warning | tail -12
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${L}_parity.log 2>&1; echo "parity_rc=$?"; tail -3 gpurun_out/${L}_parity.log
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${L}_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${L}_ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
python tools/launch_shares.py gpurun_out/${L}_launches.csv > gpurun_out/${L}_shares.json; head -c 4000 gpurun_out/${L}_shares.json
