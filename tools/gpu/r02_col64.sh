# A/B of the column split's block width (64 columns default vs MTNN_COLSPLIT_COLS=32)
set -x
exec > gpurun_out/col64.log 2>&1
timeout 600 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py tests/test_range_gpu.py 2>&1 | tail -3
for v in 64 32; do MTNN_COLSPLIT_COLS=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"split_cols" python tools/ncu_target.py nn1024x4096x4096 3 2>&1 | grep -E "duration|dram__" | head -9; done
for v in 64 32 64 32; do MTNN_COLSPLIT_COLS=$v timeout 300 python tools/probes/probe_nn_split.py 2>&1 | tail -10 | sed "s/^/c$v /"; done
for v in 64 32; do MTNN_COLSPLIT_COLS=$v timeout 300 python bench.py --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'))"; done
