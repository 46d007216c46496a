# Stream-K: parity tests, per-shape A/B, sweep A/B, FCN bench under both settings.
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "StreamK or CtaPair" 2>&1 | tail -3
timeout 900 python tools/probes/probe_streamk.py sweep 2>&1 | tail -20
MTNN_STREAMK=0 timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('fcn sk0',round(d['value'],1),d['per_call_us'])"
MTNN_STREAMK=1 timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('fcn sk1',round(d['value'],1),d['per_call_us'])"
