# A/B: the last chroma batch held behind the last luma batch (HIVC_DEBUG=defer_small=1) vs the default order
HIVC_DEBUG=defer_small=1 timeout 900 python -m pytest tests/test_gpu_bench_pins.py -x -q 2>&1 | tail -2
one() { python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']))"; }
for i in 1 2 3; do one base; HIVC_DEBUG=defer_small=1 one defer; done 2>&1 | tee gpurun_out/ab_defer.txt
