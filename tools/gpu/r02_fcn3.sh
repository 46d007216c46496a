timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_fcn3.json 2> gpurun_out/bench_fcn3.err; tail -1 gpurun_out/bench_fcn3.err
python -c "import json;d=json.load(open('gpurun_out/bench_fcn3.json'));print(d['value'], d['ms_per_step']); print(d['per_call_us']); print(d['roofline']['achieved'], d['roofline']['timed_launches_note'])"
