timeout 300 python tools/probes/probe_l2_reread.py
for v in 1 0; do MTNN_SPLIT_STRIP=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"split_cols|colmax" python tools/ncu_target.py nn1024x4096x4096 3 2>&1 | grep -E "split_cols|colmax|duration|dram__" | head -12; done
