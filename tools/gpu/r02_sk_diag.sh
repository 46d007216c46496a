timeout 300 python tools/probes/probe_streamk_steps.py 2>&1 | tail -6
for sk in 0 2; do
MTNN_STREAMK=$sk MTNN_TC_PAIR=0 timeout 300 ncu --kernel-name regex:gemm_tc3x_kernel --launch-skip 1 --launch-count 1 --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed \
  python tools/ncu_target.py nt1024x4096x4096 2>&1 | grep -E "gemm_tc3x|duration|dram__|tensor|hit_rate|per_second|lts__t_bytes" 
done
