#!/bin/bash
# Epilogue warp counts (SA_K2T_KEYSW for key launches, SA_K2T_MATSW for matrix launches) -> phase times.
cd "$(dirname "$0")/.."
run() {
  env "$@" python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ws.log 2>&1 || { tail -3 gpurun_out/ws.log; return; }
  python - "$*" <<'PY'
import json, sys
d = json.loads([x for x in open('gpurun_out/ws.log') if x.startswith('{')][-1]); ph = d['phases_ms_rank0']
print(sys.argv[1], f"step {d['ms_per_step']:.3f} S2a {ph['S2a']:.3f} S2d {ph['S2d']:.3f} S5 {ph['S5']:.3f} gemm {ph['S5_gemm']:.3f}")
PY
}
run SA_K2T_KEYSW=8
run SA_K2T_KEYSW=12
run SA_K2T_KEYSW=16
run SA_K2T_MATSW=16
run SA_K2T_MATSW=20
run SA_K2T_MATSW=8
run SA_K2T_MATSW=12
