for pp in 1 100; do
echo "=== prepass chunks $pp"
MTNN_FS_PREPASS=$pp FS=2 SHAPES=1024x4096x4096,2048x2048x2048 timeout 120 python tools/probes/probe_trace.py 2>&1 | grep -E "^\(|tma0|stage0|mma_last|chunk_last|stores_done|split_first|split_last|chunk_wait_last|pdl_wait"
done
echo "=== presplit"
FS=0 SHAPES=1024x4096x4096,2048x2048x2048 timeout 120 python tools/probes/probe_trace.py 2>&1 | grep -E "^\(|tma0|stage0|mma_last|chunk_last|stores_done|pdl_wait"
