for p in 100 100 100 100 5000 5000 5000 5000; do python bench.py --no-e2e --no-cpu-baseline --clock-period-ms $p > gpurun_out/var.log 2>&1; python - $p <<'PY'
import json,sys
d=json.loads([x for x in open('gpurun_out/var.log') if x.startswith('{')][-1])
print(sys.argv[1], round(d['ms_per_step'],3), d['clocks'].get('samples'), round(sum(v for k,v in d['phases_ms_rank0'].items() if k in ('S1','partition_S2a_to_S4','S1_received','S5')),3))
PY
done
