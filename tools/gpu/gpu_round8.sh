# Round-1 session-3 measurement pass (current kernels): tests, smoke, the four
# bench lines, ncu captures of the hot kernels and the bench launch list.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; tail -1 gpurun_out/bench_sweep.err
timeout 600 python bench.py --workload fcn --steps 10 > gpurun_out/bench_fcn.json 2> gpurun_out/bench_fcn.err; tail -1 gpurun_out/bench_fcn.err
timeout 600 python bench.py --workload large --steps 5 --no-cpu > gpurun_out/bench_large.json 2> gpurun_out/bench_large.err; tail -1 gpurun_out/bench_large.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc3x|split_rows" -s 1 -c 2 -o gpurun_out/prof_r01s4_nt8192 python tools/ncu_target.py nt8192 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc3x|split_rows" -s 1 -c 2 -o gpurun_out/prof_r01s4_skinny python tools/ncu_target.py skinny_m128 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"transpose" -s 2 -c 1 -o gpurun_out/prof_r01s4_tr16384 python tools/ncu_target.py tr16384 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"split_cols|split_rows" -s 2 -c 2 -o gpurun_out/prof_r01s4_nn4096 python tools/ncu_target.py nn1024x4096x4096 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"skinny" -s 1 -c 1 -o gpurun_out/prof_r01s4_fcn10 python tools/ncu_target.py fcn10 0 > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01s4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
ls gpurun_out | tail -30
