for rep in 1 2; do
for cap in 4096 8192 16384; do
MTNN_PIPE_BLOCKED_MAXK=$cap timeout 300 python tools/probes/probe_e2e_maxk.py $cap
done
done
