exec > gpurun_out/skinny_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"skinny_tile" -c 1 -o gpurun_out/skinny_tile python tools/probes/probe_gemv.py
ncu -i gpurun_out/skinny_tile.ncu-rep --page details 2>&1 | grep -E "Duration|Throughput|Stall|Warp Cycles|Issued|Eligible|Active Warps|Occupancy|Registers|L1/TEX Hit|L2 Hit|Mem Busy|Max Bandwidth|Achieved" | head -50
ncu -i gpurun_out/skinny_tile.ncu-rep --page raw --csv 2>&1 | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
for n,x in zip(h,v):
    if 'smsp__average_warp_latency_issue_stalled' in n or 'smsp__pcsamp_warps_issue_stalled' in n:
        try:
            if float(x.replace(',',''))>0: print(n,x)
        except: pass
"
