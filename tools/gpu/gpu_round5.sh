timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; tail -2 gpurun_out/bench_sweep.err
timeout 600 python bench.py --workload fcn --steps 5 > gpurun_out/bench_fcn.json 2> gpurun_out/bench_fcn.err; tail -2 gpurun_out/bench_fcn.err
timeout 600 python bench.py --workload large --steps 5 --no-cpu > gpurun_out/bench_large.json 2> gpurun_out/bench_large.err; tail -2 gpurun_out/bench_large.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -2 gpurun_out/bench_ref.err
for t in nt8192 nn16384; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc3x|split_rows" -s 2 -c 2 -o gpurun_out/prof_f16_$t python tools/ncu_target.py $t 3 > gpurun_out/ncu_f16_$t.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
ls gpurun_out | head -40
