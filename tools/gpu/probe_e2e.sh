for mn in 48 8; do for ch in 16 4 64; do MTNN_PIPE_MIN_MB=$mn MTNN_PIPE_CHUNK_MB=$ch timeout 120 python tools/probes/probe_e2e.py; done; done
