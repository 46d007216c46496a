# Full ncu of the FCN's 1024x4096x4096 NT GEMM (one wave of 128 tiles), warm L2
# (cache-control none: the split just wrote the halves), with source.
MTNN_STREAMK=0 timeout 600 ncu --set full --import-source on --cache-control none --clock-control none \
  --kernel-name regex:gemm_tc3x_kernel --launch-skip 1 --launch-count 1 \
  -o gpurun_out/ncu_fcn_gemm python tools/ncu_target.py nt1024x4096x4096 > gpurun_out/ncu_fcn_gemm.log 2>&1
tail -3 gpurun_out/ncu_fcn_gemm.log
MTNN_STREAMK=0 timeout 600 ncu --set full --import-source on --cache-control none --clock-control none \
  --kernel-name regex:gemm_tc3x_kernel --launch-skip 1 --launch-count 1 \
  -o gpurun_out/ncu_nt8192 python tools/ncu_target.py nt8192 > gpurun_out/ncu_nt8192.log 2>&1
tail -1 gpurun_out/ncu_nt8192.log
