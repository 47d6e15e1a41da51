#!/bin/bash
# K2T parity subset + bench phases for the u8 and fp4 operand forms.
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/epi_tests.log 2>&1; echo "tests_rc=$?"; tail -3 gpurun_out/epi_tests.log
SA_K2T_FP4=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/epi_tests_fp4.log 2>&1; echo "tests_fp4_rc=$?"; tail -3 gpurun_out/epi_tests_fp4.log
bash scripts/bench_phases.sh i8
SA_K2T_FP4=1 bash scripts/bench_phases.sh fp4
