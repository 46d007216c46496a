# Round-2 (session 4) measurement pass: bench lines, reference arm, launch list, ncu --set full of the dominant kernels.
timeout 1200 python -m pytest -q -x -m gpu tests/ > gpurun_out/r02d_gputests.log 2>&1; tail -1 gpurun_out/r02d_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 900 python bench.py > gpurun_out/r02d_sweep.json 2> gpurun_out/r02d_sweep.err; tail -1 gpurun_out/r02d_sweep.err
timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 > gpurun_out/r02d_fcn.json 2> gpurun_out/r02d_fcn.err
timeout 600 python bench.py --workload single --steps 20 --warmup 5 > gpurun_out/r02d_single.json 2> gpurun_out/r02d_single.err
timeout 600 python bench.py --workload large --steps 5 --warmup 3 --no-cpu > gpurun_out/r02d_large.json 2> gpurun_out/r02d_large.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02d_ref.json 2> gpurun_out/r02d_ref.err
timeout 300 python bench.py --impl reference --workload single --steps 5 --warmup 3 > gpurun_out/r02d_ref_single.json 2> gpurun_out/r02d_ref_single.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r02d_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-verify > /dev/null 2>&1; wc -l gpurun_out/r02d_launches.csv
for c in "pair8192 nt8192 gemm_tc3x_pair" "fcngemm nt1024x4096x4096 gemm_tc3x_kernel" "colsplit nn1024x4096x4096 split_cols" "rowsplit nt4096 split_rows" "transpose tr16384 transpose"; do
  set -- $c
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$3 --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_r02d_$1 python tools/ncu_target.py $2 3 > gpurun_out/ncu_r02d_$1.log 2>&1; tail -1 gpurun_out/ncu_r02d_$1.log
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:skinny_stream --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_r02d_skinny python tools/ncu_target.py fcn10 0 > gpurun_out/ncu_r02d_skinny.log 2>&1; tail -1 gpurun_out/ncu_r02d_skinny.log
