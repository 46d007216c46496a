exec > gpurun_out/nnrows.log 2>&1
for i in 1 2; do
TAG=rows8 python tools/probes/probe_nn_smallk.py
TAG=rows16 MTNN_B200_LIB=build/variants/nnrows16/libmtnn_b200.so python tools/probes/probe_nn_smallk.py
TAG=rows32 MTNN_B200_LIB=build/variants/nnrows32/libmtnn_b200.so python tools/probes/probe_nn_smallk.py
done
TAG=stream timeout 300 python tools/probes/probe_skinny_tile.py
