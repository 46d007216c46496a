exec > gpurun_out/fixexit.log 2>&1
for i in 1 2 3; do
python bench.py --workload fcn --steps 30 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fcn new', round(d['value'],2), d['ms_per_step'])"
MTNN_B200_LIB=build/variants/fixold/libmtnn_b200.so python bench.py --workload fcn --steps 30 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fcn old', round(d['value'],2), d['ms_per_step'])"
done
for i in 1 2; do
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-verify 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweep new', round(d['value'],2), d['ms_per_step'], d['clocks']['sm_mhz'])"
MTNN_B200_LIB=build/variants/fixold/libmtnn_b200.so python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-verify 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweep old', round(d['value'],2), d['ms_per_step'], d['clocks']['sm_mhz'])"
done
timeout 900 python -m pytest -q -x -m gpu tests/test_range_gpu.py tests/test_kernels_gpu.py 2>&1 | tail -1
