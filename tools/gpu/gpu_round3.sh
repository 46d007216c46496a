for mode in trunc rna; do for ch in 16 8 4; do echo "== $mode chunk_kb=$ch"; MTNN_SPLIT=$mode MTNN_CHUNK_KB=$ch timeout 100 python tools/probes/probe_accum.py 2>&1 | sed -n '5p'; done; done
for mode in trunc rna; do for ch in 16 8; do echo "== perf $mode chunk $ch"; MTNN_SPLIT=$mode MTNN_CHUNK_KB=$ch timeout 200 python tools/probes/probe_kernels.py 2>&1 | grep "v1:"; done; done
