echo "== accuracy: trunc (default)"; timeout 200 python tools/probes/probe_accum.py 2>&1 | tail -12
echo "== accuracy: rna"; MTNN_SPLIT=rna timeout 200 python tools/probes/probe_accum.py 2>&1 | tail -4
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; tail -c 600 gpurun_out/bench_r01b.err
