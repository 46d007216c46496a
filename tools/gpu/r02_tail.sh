timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_range_gpu.py -q -x 2>&1 | tail -2
timeout 300 python tools/probes/probe_trace.py 2>&1 | grep -E "^\(|tma0|stage0|mma_last|chunk_last|stores_done|exit|entry|pdl_wait|prologue| 12"
timeout 600 python tools/probes/probe_streamk.py 2>&1 | tail -16
