exec > gpurun_out/skinny_tile.log 2>&1
TAG=stream timeout 300 python tools/probes/probe_skinny_tile.py
python tools/probes/probe_skinny_trace.py
timeout 600 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py 2>&1 | tail -3
