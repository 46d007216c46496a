"""Sweep total with the library's per-kernel event timing on vs off (interleaved
per case), to size the instrumentation overhead inside bench.py's timed steps."""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
E = [2 ** e for e in range(7, 15)]
shapes = [(m, n, k) for m in E for n in E for k in E]
if len(sys.argv) > 1:
    shapes = [sh for sh in shapes if 2.0 * sh[0] * sh[1] * sh[2] <= float(sys.argv[1])]
A = torch.rand(16384 * 16384, device=dev) * 2 - 1
B = torch.rand(16384 * 16384, device=dev) * 2 - 1
C = torch.empty(16384 * 16384, device=dev)
tot = {0: 0.0, 1: 0.0}
for (m, n, k) in shapes:
    ev = {0: [], 1: []}
    for rep in range(4):
        for prof in (0, 1):
            L.mtnn_profile_enable(prof)
            flush.sum(); torch.cuda._sleep(200000)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); b.record()
            if rep: ev[prof].append((a, b))
    torch.cuda.synchronize()
    L.mtnn_profile_enable(0); L.mtnn_profile_reset()
    for p in (0, 1):
        tot[p] += statistics.median(a.elapsed_time(b) for a, b in ev[p])
print("cases", len(shapes), "profile off %.2f ms, on %.2f ms" % (tot[0], tot[1]))
