python -m pytest tests/test_gpu_bench_pins.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
L=paper_2008_10273_b200/libhivc_b200.so
cp $L /tmp/new.so
for v in base new base new; do
  if [ $v = base ]; then cp ab_base.so $L; else cp /tmp/new.so $L; fi
  echo $v; HIVC_DEBUG=cg_trace python tools/level_time.py 1080x1920 2>&1 | tail -2 | head -1
done
for rep in 1 2; do for v in base new; do
  if [ $v = base ]; then cp ab_base.so $L; else cp /tmp/new.so $L; fi
  python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), 'cg', round(d['roofline']['avg_launch_us'],1))"
done; done
cp /tmp/new.so $L
