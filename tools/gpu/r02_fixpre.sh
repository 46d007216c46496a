timeout 900 python -m pytest tests/test_range_gpu.py tests/test_kernels_gpu.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in default nofix; do
  fx=1; [ $v = nofix ] && fx=0
  MTNN_FIXUP=$fx timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v fcn',round(d['value'],1))"
  MTNN_FIXUP=$fx timeout 600 python bench.py --workload single --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v single',round(d['ms_per_step']*1e3,1),'us')"
done; done
