#!/bin/bash
# Tile-order group sizes: SA_K2T_GROUP (S2d, S5) and SA_K2T_GROUP_KEYS (S2a) -> phase times.
cd "$(dirname "$0")/.."
run() {
  env "$@" python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/gs.log 2>&1 || { tail -3 gpurun_out/gs.log; return; }
  python - "$*" <<'PY'
import json, sys
d = json.loads([x for x in open('gpurun_out/gs.log') if x.startswith('{')][-1]); ph = d['phases_ms_rank0']
print(sys.argv[1], f"step {d['ms_per_step']:.3f} S2a {ph['S2a']:.3f} S2d {ph['S2d']:.3f} S5 {ph['S5']:.3f} gemm {ph['S5_gemm']:.3f}")
PY
}
run SA_K2T_GROUP_KEYS=16
for g in 10 12 14 12; do run SA_K2T_GROUP=$g; done
