# GPU validation pass: gpu tests, smoke, default bench (driver contract line)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -q -x -m gpu --durations=15 > gpurun_out/pytest_gpu.log 2>&1; tail -25 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; tail -3 gpurun_out/bench_sweep.err; cat gpurun_out/bench_sweep.json | head -c 600
