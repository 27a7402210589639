python bench.py > gpurun_out/r02k_bench_line.json 2> gpurun_out/r02k_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02k_bench_reference_line.json 2>/dev/null
for i in 1 2 3; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), d['stages_ms_per_step']['device_span'])"; done
