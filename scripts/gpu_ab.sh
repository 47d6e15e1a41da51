#!/bin/bash
# A/B of environment switches on the bench line: gpu_ab.sh LABEL "ENV1" "ENV2" ...  ("-" = no env)
cd "$(dirname "$0")/.."
L=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
for e in "$@"; do
  [ "$e" = "-" ] && ee="" || ee="$e"
  env $ee timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${L}_ab.log 2>&1
  python - gpurun_out/${L}_ab.log "$e" <<'PY'
import json,sys
try:
  l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l)
  ph=d['phases_ms_rank0']
  print('%-28s ms/step %.3f S5 %.3f S5gemm %.3f S2a %.3f S2agemm %.3f S2d %.3f S2dgemm %.3f sm %s'%(sys.argv[2],d['ms_per_step'],ph['S5'],ph['S5_gemm'],ph['S2a'],ph['S2a_gemm'],ph['S2d'],ph['S2d_gemm'],d['clocks']['sm_mhz']))
except Exception as ex: print(sys.argv[2], 'FAILED', ex); print(open(sys.argv[1]).read()[-2000:])
PY
done; done
