timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 200 python tools/probes/probe_f16s.py 2>&1 | tail -12
timeout 300 python -m paper_1702_03192_b200.sweep --out gpurun_out/sweep_r01c.csv 2> gpurun_out/sweep_r01c.log
tail -2 gpurun_out/sweep_r01c.log
