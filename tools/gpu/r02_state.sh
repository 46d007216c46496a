nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv,noheader
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; tail -1 gpurun_out/bench_sweep.err
timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 > gpurun_out/bench_fcn.json 2> gpurun_out/bench_fcn.err; tail -1 gpurun_out/bench_fcn.err
timeout 600 python bench.py --workload large --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_large.json 2> gpurun_out/bench_large.err; tail -1 gpurun_out/bench_large.err
timeout 600 python bench.py --workload single --steps 20 --warmup 5 > gpurun_out/bench_single.json 2> gpurun_out/bench_single.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.err
for f in sweep fcn large single ref; do python -c "import json;d=json.load(open('gpurun_out/bench_$f.json'));print('$f', round(d['value'],3), round(d['ms_per_step'],3), d.get('e2e',{}) and round(d['e2e']['value'],2), d.get('clocks',{}).get('sm_mhz'), d.get('verify',{}) and d['verify']['failed'])"; done
