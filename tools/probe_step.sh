for rep in 1 2 3; do
for opt in "" "pre_wait"; do
  HIVC_DEBUG=$opt python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$opt', round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), d['stages_ms_per_step']['device_span'])"
done
done
