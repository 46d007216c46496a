timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_scale_gpu.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in default prevpair; do
  if [ $v = default ]; then export MTNN_B200_LIB=$PWD/paper_1702_03192_b200/lib/libmtnn_b200.so; else export MTNN_B200_LIB=$PWD/build/variants/$v/libmtnn_b200.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v sweep',round(d['value'],1),d['clocks']['sm_mhz'])"
  timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v fcn',round(d['value'],1))"
done; done
