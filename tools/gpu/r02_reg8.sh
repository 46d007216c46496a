timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "mid_shapes" 2>&1 | tail -1
MTNN_SPLIT_REG8=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "mid_shapes" 2>&1 | tail -1
for rep in 1 2; do for r8 in 0 1; do
  MTNN_SPLIT_REG8=$r8 timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());v=list(d['per_call_us'].values());print('reg8=$r8 fcn',round(d['value'],1), 'k=784/1024 calls', v[0], v[10], v[11], v[7])"
done; done
