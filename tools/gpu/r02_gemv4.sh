timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "Gemv or mid_shapes or Random or Edge" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/gemv_x.csv python tools/probes/probe_gemv.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/gemv_x.csv | head -5
for rep in 1 2; do timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());v=list(d['per_call_us'].values());print('fcn',round(d['value'],1), 'gemv calls', v[3], v[4], v[5])"; done
