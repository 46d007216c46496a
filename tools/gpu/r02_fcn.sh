timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -m gpu -k "col_split or chunk_scales or nn or tnn" 2>&1 | tail -2
timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_fcn2.json 2> gpurun_out/bench_fcn2.err; tail -1 gpurun_out/bench_fcn2.err
python -c "import json;d=json.load(open('gpurun_out/bench_fcn2.json'));print(d['value'], d['ms_per_step']); print(d['per_call_us']); print({k:(round(v['ms'],3),v['launches_per_step']) for k,v in d['kernels'].items() if k!='source'})"
timeout 600 python tools/probes/probe_fcn_breakdown.py 2>&1 | tail -1
