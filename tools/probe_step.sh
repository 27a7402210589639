python -m pytest tests/test_gpu_bench_pins.py tests/test_gpu_parity.py tests/test_gpu_edge_sizes.py tests/test_gpu_codec_behaviour.py -x -q -m gpu > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:'tree_|mask_' --csv --log-file gpurun_out/td.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/td.csv') if l.startswith('"'))]
acc=defaultdict(list)
for r in rows:
    if r['Metric Name']=='gpu__time_duration.sum':
        acc[r['Kernel Name'].split('(')[0][-40:]].append(float(r['Metric Value'].replace(',',''))/1e3)
for k,v in acc.items(): print(f"{k:42s} n={len(v):4d} mean {sum(v)/len(v):8.2f} us max {max(v):8.2f}")
PY
for i in 1 2 3; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), d['stages_ms_per_step']['device_span'])"; done
