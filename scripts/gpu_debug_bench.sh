#!/bin/bash
# S5 GEMM time under the SA_K2T_DEBUG component switches (1 no MMA, 2 no TMA, 4 no epilogue work).
cd "$(dirname "$0")/.."
for d in 0 1 2 3 4 5 6 7; do
  SA_K2T_DEBUG=$d python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/dbg$d.log 2>&1
  python - $d <<'PY'
import json, sys
d = json.loads([x for x in open(f'gpurun_out/dbg{sys.argv[1]}.log') if x.startswith('{')][-1])
ph = d['phases_ms_rank0']
print(f"debug={sys.argv[1]} step {d['ms_per_step']:.2f} S2a {ph['S2a']:.2f} S2d {ph['S2d']:.2f} S5 {ph['S5']:.2f} gemm {ph['S5_gemm']:.2f}")
PY
done
