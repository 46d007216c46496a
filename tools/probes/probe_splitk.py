"""Per-case device time (whole call) of small/mid NT shapes under the split-K
cap in this process (env MTNN_SPLITK_MAX), for A/B runs across processes."""
import os, statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
A = torch.rand(4096 * 16384, device=dev); B = torch.rand(4096 * 16384, device=dev); C = torch.empty(4096 * 4096, device=dev)
flush = torch.ones(64 * 2**20, device=dev)
shapes = [(1024, 1024, 1024), (512, 512, 4096), (1024, 1024, 4096), (256, 1024, 8192), (2048, 1024, 2048),
          (1024, 2048, 1024), (512, 2048, 2048), (1024, 1024, 16384), (2048, 2048, 2048), (128, 512, 16384)]
tot = 0
out = []
for (m, n, k) in shapes:
    ev = []
    for rep in range(8):
        flush.sum(); torch.cuda._sleep(100000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); b.record()
        if rep >= 2: ev.append((a, b))
    torch.cuda.synchronize()
    t = statistics.median(a.elapsed_time(b) for a, b in ev) * 1e3
    tot += t
    out.append(f"{m}x{n}x{k}:{t:.1f}")
print(os.environ.get("MTNN_SPLITK_MAX", "model"), f"total {tot:.1f} us |", " ".join(out), flush=True)
