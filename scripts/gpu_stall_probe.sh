#!/bin/bash
# Where do step outliers land?  Config 3 (1.8 ms steps: the host is barely ahead of the GPU) with the
# step events created inside the timed loop (SA_BENCH_LAZY_EVENTS=1, the old behaviour) and before it.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
show() { python -c "
import sys,json
l=[x for x in open('gpurun_out/stall_tmp.log') if x.startswith('{')]
if not l: print('$1','NO LINE'); sys.exit()
d=json.loads(l[-1]); print('$1', round(d['ms_per_step'],3), d['step_ms_rank0'], d['clocks'].get('samples'))
"; }
run() { tag=$1; shift; python bench.py "$@" > gpurun_out/stall_tmp.log 2>&1; show $tag; }
for r in 1 2; do
SA_BENCH_LAZY_EVENTS=1 run cfg3_s20_lazy --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline
run cfg3_s20_pre --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline
run cfg3_s40_pre --config 3 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline
run cfg5_s20_pre --config 5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline
done
run cfg4_s20_driver --gpus 1 --steps 20 --warmup 5
