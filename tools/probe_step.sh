python -m pytest tests/test_gpu_bench_pins.py tests/test_gpu_parity.py tests/test_gpu_edge_sizes.py -x -q -m gpu 2>&1 | tail -2
L=paper_2008_10273_b200/libhivc_b200.so
cp $L /tmp/new.so
for v in base new; do
  if [ $v = base ]; then cp ab_base.so $L; else cp /tmp/new.so $L; fi
  ncu --metrics gpu__time_duration.sum,launch__grid_size -k regex:frame_kernel --csv --log-file gpurun_out/pk_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
  echo $v; python tools/p_kernel_time.py gpurun_out/pk_$v.csv
  for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), d['stages_ms_per_step']['device_span'])"; done
done
