for v in default r32; do
  if [ $v = default ]; then export MTNN_B200_LIB=$PWD/paper_1702_03192_b200/lib/libmtnn_b200.so; else export MTNN_B200_LIB=$PWD/build/variants/$v/libmtnn_b200.so; fi
  echo "=== $v"
  timeout 120 python tools/probes/probe_trace.py 2>&1 | grep -E "^\(|chunk_last|stores_issued|stores_done|tma0|producer_w0|mma_last"
  MODES=base timeout 200 python tools/probes/probe_streamk.py 2>&1 | tail -15
done
export MTNN_B200_LIB=$PWD/paper_1702_03192_b200/lib/libmtnn_b200.so
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -1
