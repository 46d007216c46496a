timeout 900 python -m pytest tests/test_api_host.py tests/test_range_gpu.py -q -x -k "host or pipeline or Host" 2>&1 | tail -2
for rep in 1 2; do
OUT=gpurun_out/e2e_new_$rep.csv timeout 600 python tools/probes/probe_e2e_cases.py 2>&1 | tail -1
MTNN_PIPE_PREFIX=-1 OUT=gpurun_out/e2e_old_$rep.csv timeout 600 python tools/probes/probe_e2e_cases.py 2>&1 | tail -1
done
