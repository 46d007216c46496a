timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "Fused" 2>&1 | tail -15
timeout 600 python tools/probes/probe_fused.py 2>&1 | tail -12
