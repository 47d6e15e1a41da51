#!/bin/bash
# Final evidence of a build: default bench line, every config's table, the launch list of one
# default step and of one config-5 step, the GEMMs' ncu --set full capture.
cd "$(dirname "$0")/.."
L=${1:-r02s7}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${L}_bench.log 2>&1; echo "bench_rc=$?"; grep '^{' gpurun_out/${L}_bench.log | tail -1 | cut -c1-400
python tools/bench_configs.py --steps 10 --warmup 5 > gpurun_out/${L}_bench_configs.log 2>&1; tail -7 gpurun_out/${L}_bench_configs.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${L}_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${L}_ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
python tools/launch_shares.py gpurun_out/${L}_launches.csv > gpurun_out/${L}_shares.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${L}_cfg5_launches.csv \
  python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu_cfg5_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -c 3 \
  -o gpurun_out/${L}_gemms python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${L}_gemms_ncu.log 2>&1
echo "ncu_full_rc=$?"
