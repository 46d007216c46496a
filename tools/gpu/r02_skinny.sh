timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -m gpu -k "skinny or short_k or Kats or identity" 2>&1 | tail -3
timeout 600 python tools/probes/probe_fcn_breakdown.py 2>&1 | tail -13
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"skinny|smallk" python tools/probes/fcn_one.py nt 1024 10 4096 2>&1 | grep -E "duration|dram" | head -4
