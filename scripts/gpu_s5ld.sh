#!/bin/bash
# S5 GEMM time vs the matrices' row stride (tools/s5_bench.py, SA_S5_LD="align,extra"), two passes
cd "$(dirname "$0")/.."
for rep in 1 2; do for l in "$@"; do
  echo "$l $(SA_S5_LD=$l timeout 180 python tools/s5_bench.py 2>&1 | tail -1)"
done; done
