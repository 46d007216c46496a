for md in nt pair; do
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed --cache-control none --clock-control none \
  --kernel-name regex:gemm_tc3x --csv --log-file gpurun_out/kscale_$md.csv python tools/probes/probe_kscale.py $md > /dev/null 2>&1
done
python - <<'P'
import csv, io
for md in ("nt", "pair"):
    t = open(f"gpurun_out/kscale_{md}.csv").read().splitlines()
    s = next(i for i, l in enumerate(t) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(l for l in t[s:] if l.startswith('"')))))
    by = {}
    for r in rows:
        by.setdefault(r["ID"], {})[r["Metric Name"]] = r["Metric Value"]
    for i, (k, v) in enumerate(sorted(by.items(), key=lambda x: int(x[0]))):
        print(md, i, v)
P
