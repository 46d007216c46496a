timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; tail -1 gpurun_out/bench_sweep.err
timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_fcn.json 2> gpurun_out/bench_fcn.err
for f in sweep fcn; do python -c "import json;d=json.load(open('gpurun_out/bench_$f.json'));print('$f', round(d['value'],3), round(d['ms_per_step'],3), d.get('e2e',{}) and round(d['e2e']['value'],2), d.get('clocks',{}).get('sm_mhz'), d.get('verify',{}) and d['verify']['failed'])"; done
