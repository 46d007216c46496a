timeout 300 ncu --set full --import-source on --clock-control none -k regex:"fixup" -s 1 -c 1 -o gpurun_out/fixup_4096 python tools/probes/fcn_one.py nt 1024 4096 4096 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"skinny" -s 1 -c 1 -o gpurun_out/skinny_10 python tools/probes/fcn_one.py nt 1024 10 4096 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fixup|skinny|sgemm|split" python tools/probes/fcn_one.py nt 1024 4096 4096 2>&1 | grep -E "^  [a-z]|duration" | head -12
ls -la gpurun_out/*.ncu-rep
