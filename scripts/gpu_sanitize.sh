#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tools/sanitize_run.py.
cd "$(dirname "$0")/.."
L=${1:-r02_sanitize}
CS=/usr/local/cuda/bin/compute-sanitizer
for run in "memcheck 1" "memcheck 0" "synccheck 1" "initcheck 1" "racecheck 1"; do
  set -- $run; tool=$1; sp=$2
  {
    SA_K2T_SPARSE=$sp timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 17 python tools/sanitize_run.py \
      > gpurun_out/${L}_${tool}_sp${sp}.log 2>&1
    echo "$tool sparse=$sp rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run ok' gpurun_out/${L}_${tool}_sp${sp}.log | tr '\n' ' ')"
  }
done
