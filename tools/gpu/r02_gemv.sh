timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -2
for rep in 1 2; do for st in 1 0; do
  MTNN_SKINNY_STAGED=$st timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());v=list(d['per_call_us'].values());print('staged=$st fcn',round(d['value'],1), 'gemv calls', v[3], v[4], v[5])"
done; done
