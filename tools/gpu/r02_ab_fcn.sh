for rep in 1 2; do
for v in default start; do
  if [ $v = default ]; then export MTNN_B200_LIB=$PWD/paper_1702_03192_b200/lib/libmtnn_b200.so; else export MTNN_B200_LIB=$PWD/build/variants/start/libmtnn_b200.so; fi
  timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v fcn',round(d['value'],1), ' '.join('%.1f'%v for v in d['per_call_us'].values()), {k:round(v['ms']*1e3,1) for k,v in d['kernels'].items() if isinstance(v,dict)})"
done
done
