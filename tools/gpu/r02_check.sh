# Round-2 state check: GPU tests, smoke, default bench line.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; tail -1 gpurun_out/bench_sweep.err; cat gpurun_out/bench_sweep.json | head -c 600
