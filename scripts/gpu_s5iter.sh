#!/bin/bash
# S5 epilogue iteration: the matrix parity tests, then the S5 GEMM time in the bench line.
cd "$(dirname "$0")/.."
L=${1:-s3b}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_matrices.py \
  "tests/test_gpu_parity.py::test_f_division_free_is_ieee_rn" "tests/test_gpu_parity.py::test_bucket_similarity_random" \
  "tests/test_gpu_parity.py::test_bucket_similarity_batch" > gpurun_out/${L}_tests.log 2>&1
echo "tests_rc=$?"; tail -3 gpurun_out/${L}_tests.log
for i in 1 2; do
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/${L}_bench$i.log 2>&1; echo "bench_rc=$?"
python - gpurun_out/${L}_bench$i.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l)
ph=d['phases_ms_rank0']; r=d['roofline']
print('ms/step %.3f S5 %.3f S5gemm %.3f S2a %.3f S2agemm %.3f S2d %.3f frac_hbm %.3f clocks %s'%(d['ms_per_step'],ph['S5'],ph['S5_gemm'],ph['S2a'],ph['S2a_gemm'],ph['S2d'],r['frac_hbm'],d['clocks']))
PY
done
