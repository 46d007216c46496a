exec > gpurun_out/stages.log 2>&1
for i in 1 2; do
TAG=base python tools/probes/probe_inkernel_stages.py
TAG=hl4raw5 MTNN_B200_LIB=build/variants/hl4raw5/libmtnn_b200.so python tools/probes/probe_inkernel_stages.py
TAG=hl4raw4 MTNN_B200_LIB=build/variants/hl4raw4/libmtnn_b200.so python tools/probes/probe_inkernel_stages.py
done
MTNN_B200_LIB=build/variants/hl4raw5/libmtnn_b200.so timeout 600 compute-sanitizer --tool racecheck python tools/probes/race_one.py 128 2048 256 2>&1 | grep SUMMARY
MTNN_B200_LIB=build/variants/hl4raw5/libmtnn_b200.so timeout 900 python -m pytest -q -x -m gpu tests/test_range_gpu.py tests/test_kernels_gpu.py 2>&1 | tail -1
