# r02n: GPU tests, bench line + repeats, reference arm, launch list of the bench command (final tree of round 2)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/r02n_gputest.txt; cat gpurun_out/r02n_gputest.txt
python bench.py > gpurun_out/r02n_bench_line.json 2> gpurun_out/r02n_bench.err
for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']))"; done | tee gpurun_out/r02n_repeats.txt
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02n_bench_reference_line.json 2> gpurun_out/r02n_ref.err; cut -c1-300 gpurun_out/r02n_bench_reference_line.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02n_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02n_launches_bench.csv > gpurun_out/r02n_launches_summary.txt 2>&1; head -14 gpurun_out/r02n_launches_summary.txt
