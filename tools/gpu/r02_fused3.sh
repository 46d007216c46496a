for v in default diag1 diag2; do
  if [ $v = default ]; then export MTNN_B200_LIB=$PWD/paper_1702_03192_b200/lib/libmtnn_b200.so; else export MTNN_B200_LIB=$PWD/build/variants/$v/libmtnn_b200.so; fi
  echo "=== $v"
  FS=2 SHAPES=1024x4096x4096 timeout 120 python tools/probes/probe_trace.py 2>&1 | grep -E "^\(|stage0|mma_last|stores_done|split_first|split_last|chunk_wait_last"
done
