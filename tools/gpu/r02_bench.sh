# bench contract tests + default bench + single/fcn/reference lines
nproc; nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv,noheader
timeout 1200 python -m pytest tests/test_bench_contract.py -q -x -m gpu 2>&1 | tail -5
timeout 900 python bench.py > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; tail -2 gpurun_out/bench_sweep.err
timeout 600 python bench.py --workload single --steps 20 --warmup 5 > gpurun_out/bench_single.json 2> gpurun_out/bench_single.err; tail -1 gpurun_out/bench_single.err
timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 > gpurun_out/bench_fcn.json 2> gpurun_out/bench_fcn.err; tail -1 gpurun_out/bench_fcn.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.err
timeout 300 python bench.py --impl reference --workload single --steps 5 --warmup 1 > gpurun_out/bench_ref_single.json 2> gpurun_out/bench_ref_single.err
