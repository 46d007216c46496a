"""Sustained A/B of single-CTA vs CTA-pair tiles on the large config (65536 x
8192 x 8192): blocks of back-to-back launches alternating the tc_pair knob,
with nvidia-smi clock/power samples per block."""
import statistics, subprocess, sys, threading, time, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
m, n, k = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (65536, 8192, 8192))]
A = torch.rand(m * k, device=dev) * 2 - 1; B = torch.rand(n * k, device=dev) * 2 - 1; C = torch.empty(m * n, device=dev)
samples = []
stop = threading.Event()
def sampler():
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line: samples.append((time.time(), *[float(x) for x in line.split(",")]))
    p.terminate()
th = threading.Thread(target=sampler); th.start()
res = {0: [], 1: []}
for blk in range(8):
    mode = blk % 2
    _lib.config_set("tc_pair", 2 * mode)  # 0 = single-CTA tiles, 2 = pairs forced
    _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); torch.cuda.synchronize()
    t0 = time.time()
    ev = []
    for i in range(25):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    t1 = time.time()
    ms = statistics.median(x.elapsed_time(y) for x, y in ev)
    cl = [c for (t, c, p) in samples if t0 <= t <= t1]; pw = [p for (t, c, p) in samples if t0 <= t <= t1]
    res[mode].append(ms)
    print(f"block {blk} pair={mode}: {ms:.3f} ms {2*m*n*k/ms/1e9:.0f} TF/s clock {statistics.median(cl) if cl else 0:.0f} MHz power {statistics.median(pw) if pw else 0:.0f} W", flush=True)
stop.set(); th.join()
for mode in (0, 1):
    print("pair", mode, "median ms", statistics.median(res[mode]))
