for rep in 1 2; do for fx in 1 0; do
  MTNN_FIXUP=$fx timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('fixup=$fx sweep',round(d['value'],1),d['clocks']['sm_mhz'])"
  MTNN_FIXUP=$fx timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('fixup=$fx fcn',round(d['value'],1), ' '.join('%.1f'%v for v in d['per_call_us'].values()))"
  MTNN_FIXUP=$fx timeout 600 python bench.py --workload single --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('fixup=$fx single',round(d['ms_per_step']*1e3,1),'us')"
done; done
