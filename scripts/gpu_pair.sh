#!/bin/bash
# CTA-pair K2T bring-up: quick parity subset under a hard timeout, then the full GPU suite and phases.
cd "$(dirname "$0")/.."
timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "bucket_similarity_batch" > gpurun_out/pair_quick.log 2>&1; rc=$?
echo "quick_rc=$rc"; tail -3 gpurun_out/pair_quick.log
[ $rc -ne 0 ] && exit 1
bash scripts/gpu_check.sh
bash scripts/gpu_k2t_debug.sh 2>&1 | sed -n '1p;5p;7p;8p'
