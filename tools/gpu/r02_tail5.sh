timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_range_gpu.py tests/test_scale_gpu.py -q -x 2>&1 | tail -1
MTNN_B200_LIB=build/variants/trace/libmtnn_b200.so FS=0 SHAPES=1024x4096x4096,1024x1024x1024 timeout 120 python tools/probes/probe_trace.py 2>&1 | grep -E "^\(|chunk_last|last_promoted|first_store|stores_issued|stores_done"
for rep in 1 2; do for v in default nodirect; do
  if [ $v = default ]; then export MTNN_B200_LIB=$PWD/paper_1702_03192_b200/lib/libmtnn_b200.so; else export MTNN_B200_LIB=$PWD/build/variants/$v/libmtnn_b200.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v sweep',round(d['value'],1),d['clocks']['sm_mhz'])"
  timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v fcn',round(d['value'],1))"
  timeout 600 python bench.py --workload single --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v single',round(d['ms_per_step']*1e3,1),'us')"
done; done
