"""Fixed-cost probe: small/mid shapes per variant (profiling off, median of 7,
L2 flushed, GPU kept busy by a spin kernel ahead of each window)."""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
import os
N2 = 16384 * 16384 if os.environ.get('LONGSKINNY') else 4096 * 4096
A = torch.rand(N2, device=dev); B = torch.rand(N2, device=dev); C = torch.empty(N2, device=dev)
import os
shapes = [(128, 128, 128), (256, 128, 128), (128, 1024, 256), (512, 512, 512), (1024, 1024, 256), (256, 2048, 512),
          (1024, 1024, 1024), (2048, 2048, 512), (512, 4096, 1024), (2048, 2048, 2048)]
if os.environ.get("TINY"):
    shapes = [(32, 32, 32), (64, 64, 64), (64, 64, 256), (128, 128, 64), (128, 128, 128), (96, 200, 128), (256, 256, 32), (128, 64, 512)]
if os.environ.get("LONGSKINNY"):
    shapes = [(128, 16384, 16384), (16384, 128, 16384), (256, 16384, 16384), (128, 16384, 4096), (256, 8192, 8192), (512, 16384, 16384), (128, 4096, 16384)]
if os.environ.get("SKINNY"):
    shapes = [(m, n, k) for m in (128, 256, 512) for n in (128, 256, 512, 2048) for k in (128, 512, 2048)]
names = {0: "auto", 1: "tf32", 2: "ffma", 3: "f16s"}
for (m, n, k) in shapes:
    out = []
    for v in (2, 1, 3, 0):
        ev = []
        for rep in range(8):
            flush.sum(); torch.cuda._sleep(100000)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, v, s)); b.record()
            if rep: ev.append((a, b))
        torch.cuda.synchronize()
        t = statistics.median(a.elapsed_time(b) for a, b in ev) * 1e3
        out.append(f"{names[v]} {t:6.1f}us")
    print(f"({m},{n},{k}) " + "  ".join(out), flush=True)
