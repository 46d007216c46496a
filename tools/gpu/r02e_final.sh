# Round-2 session-4 closing pass: GPU suite, smoke, the default bench line (sweep) and the FCN line.
timeout 1200 python -m pytest -q -x -m gpu tests/ > gpurun_out/r02e_gputests.log 2>&1; tail -1 gpurun_out/r02e_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02e_sweep.json 2> gpurun_out/r02e_sweep.err; tail -1 gpurun_out/r02e_sweep.err
timeout 600 python bench.py --workload fcn --steps 20 --warmup 5 > gpurun_out/r02e_fcn.json 2> gpurun_out/r02e_fcn.err
timeout 600 python bench.py --workload single --steps 20 --warmup 5 > gpurun_out/r02e_single.json 2> gpurun_out/r02e_single.err
