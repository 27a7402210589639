nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02m_gputest.txt
cat gpurun_out/r02m_gputest.txt
python bench.py > gpurun_out/r02m_bench_line.json 2> gpurun_out/r02m_bench.err
tail -c 600 gpurun_out/r02m_bench_line.json
