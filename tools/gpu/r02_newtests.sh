timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_range_gpu.py -q -x -k "gate or pipelined_matches or host_pipelines" 2>&1 | tail -3
