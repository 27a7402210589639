python -m pytest tests/test_gpu_bench_pins.py tests/test_gpu_parity.py tests/test_gpu_edge_sizes.py tests/test_gpu_codec_behaviour.py -x -q -m gpu > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
L=paper_2008_10273_b200/libhivc_b200.so
cp $L /tmp/new.so
for rep in 1 2 3; do
for v in base new; do
  if [ $v = base ]; then cp ab_base.so $L; else cp /tmp/new.so $L; fi
  HIVC_DEBUG=p_repeat=4 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), d['stages_ms_per_step']['device_span'])"
done
done
cp /tmp/new.so $L
