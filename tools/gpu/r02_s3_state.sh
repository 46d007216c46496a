# Session-3 state on a fresh build: GPU tests, smoke, all bench lines, launch list.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/gpu/r02_state.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_fcn.csv python bench.py --workload fcn --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1; wc -l gpurun_out/launches_fcn.csv
