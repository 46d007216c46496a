timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -m gpu -k "skinny or short_k or Kats or identity" 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"skinny" python tools/probes/fcn_one.py nt 1024 10 4096 2>&1 | grep -E "duration|dram" | head -4
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"skinny" python tools/probes/fcn_one.py nt 10 4096 1024 2>&1 | grep -E "duration|dram" | head -4
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:"sgemm" python tools/probes/fcn_one.py nn 1024 4096 10 2>&1 | grep -E "duration|dram" | head -4
timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_fcn4.json 2> gpurun_out/bench_fcn4.err; tail -1 gpurun_out/bench_fcn4.err
python -c "import json;d=json.load(open('gpurun_out/bench_fcn4.json'));print(d['value'], d['ms_per_step']); print(d['per_call_us'])"
