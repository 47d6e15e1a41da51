#!/bin/bash
# env A/B: S5-only timing (tools/s5_bench.py) and bench lines, alternating, for each env setting given
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do for s in "$@"; do
  case $s in DEF) e="";; *) e="$s";; esac
  echo "s5 $s $(env $e timeout 180 python tools/s5_bench.py 2>&1 | tail -1)"
done; done
[ -n "$NOBENCH" ] && exit 0
for rep in $(seq ${REPS:-2}); do for s in "$@"; do
  case $s in DEF) e="";; *) e="$s";; esac
  env $e timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/envab_b.log 2>&1
  python - gpurun_out/envab_b.log "$s" <<'PY'
import json,sys
try:
  l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l)
  ph=d['phases_ms_rank0']
  print('bench %-16s ms/step %.3f S5 %.3f S5gemm %.3f S2a %.3f S2agemm %.3f S2d %.3f S2dgemm %.3f sm %s'%(sys.argv[2],d['ms_per_step'],ph['S5'],ph['S5_gemm'],ph['S2a'],ph['S2a_gemm'],ph['S2d'],ph['S2d_gemm'],d['clocks']['sm_mhz']))
except Exception as ex: print(sys.argv[2], 'FAILED', ex); print(open(sys.argv[1]).read()[-1500:])
PY
done; done
