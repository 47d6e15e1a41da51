#!/bin/bash
# SA_SCRATCH_CACHE=1 (library-kept large scratch blocks): config 3's tenth-step outlier with and without it,
# config 4 both ways, then the whole GPU suite with the cache on.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
one() { tag=$1; shift; "$@" > gpurun_out/sc_tmp.log 2> gpurun_out/sc_tmp.err
python -c "
import json
l=[x for x in open('gpurun_out/sc_tmp.log') if x.startswith('{')]
if not l: print('$tag NO LINE'); print(open('gpurun_out/sc_tmp.err').read()[-1500:]); raise SystemExit
d=json.loads(l[-1]); print('$tag', round(d['ms_per_step'],3), [round(x,2) for x in d['step_ms_rank0']])
"; grep "held the host" gpurun_out/sc_tmp.err | tail -3; }
for r in 1 2; do
one cfg3_off env SA_TRACE_ALLOC=1 python bench.py --config 3 --steps 12 --warmup 5 --no-e2e --no-cpu-baseline
one cfg3_on env SA_TRACE_ALLOC=1 SA_SCRATCH_CACHE=1 python bench.py --config 3 --steps 12 --warmup 5 --no-e2e --no-cpu-baseline
done
one cfg4_on env SA_SCRATCH_CACHE=1 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline
one cfg4_off python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline
one cfg5_on env SA_SCRATCH_CACHE=1 python bench.py --config 5 --steps 12 --warmup 5 --no-e2e --no-cpu-baseline
SA_SCRATCH_CACHE=1 timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/sc_tests.log 2>&1; echo "tests_rc(cache on)=$?"; tail -1 gpurun_out/sc_tests.log
