#!/bin/bash
# Config 3's tenth-step outlier under the ncu launch list: per-kernel durations of every launch of
# 12 timed steps -- a kernel of S2a that stretches in step 10 shows as an outlier among its own launches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/stall3_launches.csv \
  python bench.py --config 3 --steps 12 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/stall3.log 2>&1; echo "rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/stall3_launches.csv')))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; kn = h.index('Kernel Name'); mv = h.index('Metric Value')
by = collections.defaultdict(list)
for i, r in enumerate(rows[hi + 2:]):
    if len(r) > mv:
        by[r[kn][:50]].append((float(r[mv].replace(',', '')) / 1000, i))
for k, v in by.items():
    if len(v) < 8: continue
    d = sorted(x for x, _ in v); med = d[len(d) // 2]
    out = [(round(x, 1), i) for x, i in v if x > 3 * med + 20]
    if out: print(k, 'median us', round(med, 1), 'outliers (us, launch index)', out[:6])
print('kernels', sum(len(v) for v in by.values()))
l = [x for x in open('gpurun_out/stall3.log') if x.startswith('{')]
if l:
    import json; d = json.loads(l[-1]); print('S2a per step (under ncu)', d['phase_steps_ms_rank0']['S2a'])
PY
