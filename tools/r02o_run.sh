# r02o: GPU tests, bench line + repeats, reference arm, launch list of the bench command (final tree of round 2)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/r02o_gputest.txt; cat gpurun_out/r02o_gputest.txt
python bench.py > gpurun_out/r02o_bench_line.json 2> gpurun_out/r02o_bench.err
for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']))"; done | tee gpurun_out/r02o_repeats.txt
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02o_bench_reference_line.json 2> gpurun_out/r02o_ref.err; cut -c1-300 gpurun_out/r02o_bench_reference_line.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02o_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02o_launches_bench.csv > gpurun_out/r02o_launches_summary.txt 2>&1; head -14 gpurun_out/r02o_launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cg_tile_kernel -s 20 -c 1 -o gpurun_out/r02o_cg_tile_bench python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/r02o_ncu_cg.log 2>&1; tail -2 gpurun_out/r02o_ncu_cg.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum -k regex:'cg_tile|cg_cluster|frame_kernel|restrict|cg_setup' --clock-control none --csv --log-file gpurun_out/r02o_km.csv python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/ncu_kernel_summary.py gpurun_out/r02o_km.csv --out gpurun_out/r02o_kernel_metrics.json > gpurun_out/r02o_km.err 2>&1; head -c 400 gpurun_out/r02o_kernel_metrics.json
