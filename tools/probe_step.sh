python -m pytest tests/test_gpu_bench_pins.py tests/test_gpu_parity.py tests/test_gpu_edge_sizes.py -x -q -m gpu > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
ncu --metrics gpu__time_duration.sum,launch__grid_size --cache-control none --clock-control none -k regex:'restrict|setup' --csv --log-file gpurun_out/setup_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/setup_launches.csv') if l.startswith('"'))]
by=defaultdict(dict)
for r in rows: by[(int(r['ID']),r['Kernel Name'][:40])][r['Metric Name']]=float(r['Metric Value'].replace(',',''))
last=sorted(by.items())[-len(by)//2:]
tot=0
for (i,n),m in last:
    tot+=m['gpu__time_duration.sum']/1e3
    print(f"{i:5d} {n:40s} grid {int(m.get('launch__grid_size',0)):7d} {m['gpu__time_duration.sum']/1e3:8.2f} us")
print("total", tot)
PY
cat gpurun_out/pt.log | tail -2
python - <<PY
print()
PY
for i in 1 2 3; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), d['stages_ms_per_step']['device_span'])"; done
