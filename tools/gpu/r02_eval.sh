timeout 600 python tools/probes/probe_fcn_breakdown.py 2>&1 | tail -14
timeout 1200 python -m pytest tests/test_reference_suite_gpu.py -q -x -s 2>&1 | tail -15
timeout 1500 python tools/eval_report.py --out gpurun_out/eval_r02 2>&1 | tail -12
timeout 900 python tools/ref_vs_port.py gpurun_out/ref_vs_port.json > /dev/null 2>&1; tail -30 gpurun_out/ref_vs_port.json
