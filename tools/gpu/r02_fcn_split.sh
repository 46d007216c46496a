exec > gpurun_out/fcn_split.log 2>&1
python tools/probes/probe_fcn_breakdown.py
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fcn_launches.csv python tools/probes/fcn_calls_once.py
