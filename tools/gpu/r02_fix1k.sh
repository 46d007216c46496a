exec > gpurun_out/fix1k.log 2>&1
for i in 1 2; do
python tools/probes/probe_fcn_breakdown.py | tail -1 | sed 's/^/base /'
MTNN_B200_LIB=build/variants/fix1k/libmtnn_b200.so python tools/probes/probe_fcn_breakdown.py | tail -1 | sed 's/^/fix1k /'
python bench.py --workload fcn --steps 20 --warmup 5 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench base', d['value'], d['ms_per_step'])"
MTNN_B200_LIB=build/variants/fix1k/libmtnn_b200.so python bench.py --workload fcn --steps 20 --warmup 5 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench fix1k', d['value'], d['ms_per_step'])"
done
