CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_memcheck.txt 2>&1; tail -4 gpurun_out/san_memcheck.txt
MTNN_F16S_INKERNEL=0 timeout 1500 $CS --tool racecheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_racecheck.txt 2>&1; tail -4 gpurun_out/san_racecheck.txt
MTNN_F16S_INKERNEL=0 timeout 1500 $CS --tool synccheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_synccheck.txt 2>&1; tail -4 gpurun_out/san_synccheck.txt
