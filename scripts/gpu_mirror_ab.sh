#!/bin/bash
# A/B of the mirrored-store experiment builds (SA_MIRROR_V2 / SA_MIRROR_LAST, scripts/build_variant.sh)
# against lib/libsa.so: S5 GEMM + bench line alternating, then the matrix parity tests on each variant.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=mirror bash scripts/gpu_libab.sh "$@"
for v in "$@"; do
  [ "$v" = "-" ] && continue
  SA_LIBSA=paper_0905_1744_b200/lib/libsa_$v.so timeout 600 python -m pytest -q -m gpu -x tests/test_gpu_matrices.py \
    "tests/test_gpu_parity.py::test_bucket_similarity_random" "tests/test_gpu_parity.py::test_bucket_similarity_batch" \
    > gpurun_out/mirror_tests_$v.log 2>&1
  echo "$v tests_rc=$? $(tail -1 gpurun_out/mirror_tests_$v.log)"
done
for r in 1 2; do python tools/tree_bench.py --buckets 8 2>&1 | tail -1; done
