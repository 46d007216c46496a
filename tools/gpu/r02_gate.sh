timeout 900 python -m pytest tests/test_bench_contract.py -q -x -m gpu 2>&1 | tail -2
for rep in 1 2 3 4; do
  timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('fcn',round(d['value'],1),round(d['wall_ms_per_step'],3))"
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('sweep',round(d['value'],1),d['clocks']['sm_mhz'])"
timeout 600 python bench.py --workload single --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('single',round(d['value'],2),round(d['ms_per_step']*1e3,1),'us')"
