exec > gpurun_out/reduce4.log 2>&1
timeout 900 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py tests/test_range_gpu.py 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk_reduce" python tools/probes/fcn_calls_once.py 2>&1 | grep -E "splitk|duration"
python tools/probes/probe_fcn_breakdown.py | tail -3
