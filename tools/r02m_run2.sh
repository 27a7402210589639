# r02m: GPU tests (incl. the wrapper goldens), bench repeats, launch list, full captures of the two top kernels
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/r02m_gputest.txt; cat gpurun_out/r02m_gputest.txt
python bench.py > gpurun_out/r02m_bench_line.json 2> gpurun_out/r02m_bench.err
for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']))"; done | tee gpurun_out/r02m_repeats.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02m_launches_bench.csv > gpurun_out/r02m_launches_summary.txt 2>&1; head -14 gpurun_out/r02m_launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cg_tile_kernel -s 20 -c 1 -o gpurun_out/r02m_cg_tile_bench python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/r02m_ncu_cg.log 2>&1; tail -2 gpurun_out/r02m_ncu_cg.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 400 -c 1 -o gpurun_out/r02m_frame_kernel_bench python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/r02m_ncu_fk.log 2>&1; tail -2 gpurun_out/r02m_ncu_fk.log
