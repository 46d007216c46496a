for t in 0 1 2; do
echo "== tail $t"
MTNN_B200_LIB=build/variants/trace_t$t/libmtnn_b200.so FS=0 SHAPES=1024x4096x4096,1024x1024x1024 timeout 120 python tools/probes/probe_trace.py 2>&1 | grep -E "^\(|chunk_last|last_promoted|first_store|stores_issued|stores_done"
done
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -1
for rep in 1 2; do for t in 0 1 2; do
MTNN_B200_LIB=build/variants/tail$t/libmtnn_b200.so timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('tail$t fcn',round(d['value'],1))"
MTNN_B200_LIB=build/variants/tail$t/libmtnn_b200.so timeout 600 python bench.py --workload single --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('tail$t single',round(d['ms_per_step']*1e3,1),'us')"
done; done
