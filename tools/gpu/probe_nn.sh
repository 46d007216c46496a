for cfg in 2048,512,1024,0,1 512,2048,1024,0,1 2048,1024,1024,0,1; do MTNN_DEBUG_NN=$cfg timeout 60 python tools/probes/probe_nn.py; done
