#!/bin/bash
# K2T component switches on one aligned cfg4-shaped bucket (tools/k2_bench.py; never the full pipeline:
# garbage keys would send sa_partition to its exact host fallback).  Columns: S5 matrices, sym keys, rect keys:
# [whole call ms, GEMM-only ms].  SA_K2T_DEBUG bits: 1 no MMA, 2 no TMA, 4 no epilogue, 8 no matrix stores.
cd "$(dirname "$0")/.."
N=${N:-12544}
for d in ${DBG:-0 1 2 3 4 5 6 7 8}; do
  echo "debug=$d $(SA_K2T_DEBUG=$d timeout 120 python tools/k2_bench.py --n $N 2>&1 | grep -v engine | python3 -c "import sys,json; print([(round(json.loads(l)['ms'],3), round(json.loads(l)['gemm_ms'],3)) for l in sys.stdin if l.startswith('{')])")"
done
