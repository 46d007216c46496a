for rep in 1 2; do
timeout 120 python tools/probes/probe_splitk.py
for c in 1 2 4; do MTNN_SPLITK_MAX=$c timeout 120 python tools/probes/probe_splitk.py; done
done
