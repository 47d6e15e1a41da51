#!/bin/bash
# S5 GEMM DRAM read/write bytes under store switches (where do the extra reads come from?):
# time by tools/s5_bench.py, bytes by one ncu launch of the same call.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum
for s in "${@:-DEF}"; do
  case $s in DEF) e="";; *) e="$s";; esac
  [ -n "$NOTIME" ] || t=$(env $e timeout 180 python tools/s5_bench.py 2>&1 | tail -1)
  env $e timeout 300 ncu --metrics $M --clock-control none -k regex:gemm2 -c 1 --csv \
    python tools/s5_bench.py --once > gpurun_out/s5dram_$$.csv 2>/dev/null
  echo "== $s :: $t"
  grep -E '"(gpu__time|dram__|lts__)' gpurun_out/s5dram_$$.csv | awk -F'","' '{print "   ",$(NF-2),$(NF-1),$NF}'
done
