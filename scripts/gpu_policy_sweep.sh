#!/bin/bash
# Operand L2 policies of the CTA-pair K2T GEMM (SA_K2T_EVICT_LAST bits: 1/2 A/B evict_last, 4/8 A/B evict_first).
cd "$(dirname "$0")/.."
for v in 0 1 8 9 2 3 12 4 0; do
  SA_K2T_EVICT_LAST=$v python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ps.log 2>&1 || { tail -3 gpurun_out/ps.log; continue; }
  python - "$v" <<'PY'
import json, sys
d = json.loads([x for x in open('gpurun_out/ps.log') if x.startswith('{')][-1]); ph = d['phases_ms_rank0']
print("policy", sys.argv[1], f"step {d['ms_per_step']:.3f} S2a {ph['S2a']:.3f} S2d {ph['S2d']:.3f} S5 {ph['S5']:.3f} gemm {ph['S5_gemm']:.3f}")
PY
done
