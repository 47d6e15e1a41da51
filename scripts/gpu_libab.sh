#!/bin/bash
# A/B of library builds (lib/libsa_NAME.so; "-" = lib/libsa.so) in one call:
# S5 GEMM alone (tools/s5_bench.py) and the bench line, alternating.
#   TESTS=1 runs the matrix parity tests on lib/libsa.so first.
cd "$(dirname "$0")/.."
L=${L:-ab}
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_matrices.py \
    "tests/test_gpu_parity.py::test_f_division_free_is_ieee_rn" "tests/test_gpu_parity.py::test_bucket_similarity_random" \
    "tests/test_gpu_parity.py::test_bucket_similarity_batch" $TESTS_EXTRA > gpurun_out/${L}_tests.log 2>&1
  echo "tests_rc=$?"; tail -2 gpurun_out/${L}_tests.log
fi
for rep in 1 2; do
for v in "$@"; do
  [ "$v" = "-" ] && lib="" || lib="paper_0905_1744_b200/lib/libsa_$v.so"
  echo "$v s5: $(SA_LIBSA=$lib timeout 180 python tools/s5_bench.py 2>&1 | tail -1)"
  SA_LIBSA=$lib timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/${L}_b.log 2>&1
  python - gpurun_out/${L}_b.log "$v" <<'PY'
import json,sys
try:
  l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l)
  ph=d['phases_ms_rank0']
  print('%-8s bench ms/step %.3f S5 %.3f S5gemm %.3f S2a %.3f S2agemm %.3f S2d %.3f S2dgemm %.3f sm %s'%(sys.argv[2],d['ms_per_step'],ph['S5'],ph['S5_gemm'],ph['S2a'],ph['S2a_gemm'],ph['S2d'],ph['S2d_gemm'],d['clocks']['sm_mhz']))
except Exception as ex: print(sys.argv[2], 'FAILED', ex); print(open(sys.argv[1]).read()[-1500:])
PY
done; done
