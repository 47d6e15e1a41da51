#!/bin/bash
# Bench-line A/B of library builds (lib/libsa_NAME.so; "-" = lib/libsa.so), alternating, no S5-only runs.
cd "$(dirname "$0")/.."
L=${L:-ab}
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest -q -m gpu -x $TESTS > gpurun_out/${L}_tests.log 2>&1
  echo "tests_rc=$?"; tail -2 gpurun_out/${L}_tests.log
fi
for rep in $(seq ${REPS:-2}); do
for v in "$@"; do
  [ "$v" = "-" ] && lib="" || lib="paper_0905_1744_b200/lib/libsa_$v.so"
  SA_LIBSA=$lib timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${L}_b.log 2>&1
  python - gpurun_out/${L}_b.log "$v" <<'PY'
import json,sys
try:
  l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l)
  ph=d['phases_ms_rank0']
  print('%-6s ms/step %.3f S1 %.3f S1r %.3f S5 %.3f S5gemm %.3f S2a %.3f S2agemm %.3f S2d %.3f S2dgemm %.3f S3 %.3f sm %s'%(sys.argv[2],d['ms_per_step'],ph['S1'],ph['S1_received'],ph['S5'],ph['S5_gemm'],ph['S2a'],ph['S2a_gemm'],ph['S2d'],ph['S2d_gemm'],ph['S3'],d['clocks']['sm_mhz']))
except Exception as ex: print(sys.argv[2], 'FAILED', ex); print(open(sys.argv[1]).read()[-1500:])
PY
done; done
