#!/bin/bash
# S5 GEMM under SA_K2T_DEBUG switches (tools/s5_bench.py: the bench's 8 config-4 buckets, one launch).
# bits: 1 no MMA, 2 no TMA loads, 8 no matrix stores, 64 F stand-in (no fp64), 128 no column tables,
# 256 no corrections, 512 no mirrored stores, 1024 no C stores, 2048 no C packing,
# 4096 no direct-half staging / TMA stores, 8192 TMEM loads only (no chunk work); 4 no chunk loop at all
cd "$(dirname "$0")/.."
for d in ${DBG:-0}; do
  for ee in ${ENVS:--}; do
    [ "$ee" = "-" ] && e2="" || e2="$ee"
    echo "$ee $(env $e2 SA_K2T_DEBUG=$d timeout 180 python tools/s5_bench.py 2>&1 | tail -1)"
  done
done
