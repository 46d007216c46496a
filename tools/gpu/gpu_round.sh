set -x
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -c 3000 gpurun_out/bench_r01.json
timeout 300 python -m paper_1702_03192_b200.sweep --out gpurun_out/sweep_auto2.csv 2> gpurun_out/sweep_auto2.log
for t in nt8192 nt16384 nn16384 tr16384; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc3xtf32|transpose_vec4" -s 1 -c 1 -o gpurun_out/prof_$t python tools/ncu_target.py $t > gpurun_out/ncu_$t.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
ls -la gpurun_out
