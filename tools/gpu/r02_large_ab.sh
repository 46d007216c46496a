exec > gpurun_out/large_ab.log 2>&1
for i in 1 2; do
for lib in new old; do
  if [ $lib = old ]; then export MTNN_B200_LIB=build/wt_s4/paper_1702_03192_b200/lib/libmtnn_b200.so; else unset MTNN_B200_LIB; fi
  timeout 600 python bench.py --workload large --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
