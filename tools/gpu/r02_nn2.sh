timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -m gpu -k "col_split or chunk_scales or nn" 2>&1 | tail -2
timeout 600 python tools/probes/probe_fcn_breakdown.py 2>&1 | grep -E "^nn|total"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_tc3x" python tools/ncu_target.py nn1024x4096x4096 3 2>&1 | grep -E "duration" | head -4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_tc3x|split" python tools/ncu_target.py nn16384 3 2>&1 | grep -E "duration|split_c|pair" | head -12
