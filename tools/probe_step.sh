python -m pytest tests/test_gpu_bench_pins.py tests/test_gpu_parity.py tests/test_gpu_edge_sizes.py -x -q -m gpu > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
HIVC_DEBUG=cg_trace python tools/level_time.py 1080x1920 2>&1 | tail -2 | head -1
for i in 1 2 3; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']))"; done
