timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -4
timeout 600 python tools/probes/probe_fcn_breakdown.py 2>&1 | tail -14
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"split_cols|gemm_tc3x" python tools/ncu_target.py nn1024x4096x4096 3 2>&1 | grep -E "split_cols|gemm_tc3x|duration|dram__" | head -12
