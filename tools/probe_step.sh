# r02l: final bench line and launch list on the current tree
python bench.py > gpurun_out/r02l_bench_line.json 2> gpurun_out/r02l_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02l_launches_bench.csv > gpurun_out/r02l_launches_summary.txt 2>&1; head -12 gpurun_out/r02l_launches_summary.txt
HIVC_DEBUG=cg_trace python tools/level_time.py 1080x1920 2>&1 | tail -2 | head -1
for i in 1 2 3; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']))"; done
