timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -2
for st in 1 0; do
MTNN_SKINNY_STAGED=$st timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/gemv_$st.csv python tools/probes/probe_gemv.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/gemv_$st.csv | head -6
done
