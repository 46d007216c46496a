"""Row split at k = 1024 (A/B with MTNN_SPLIT_REG1024): ncu-free device time of
NT calls whose splits are k = 1024 rows, plus the split-class time."""
import os, statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device="cuda")
A = torch.rand(16384 * 16384, device="cuda"); B = torch.rand(16384 * 16384, device="cuda"); C = torch.empty(16384 * 16384, device="cuda")
tag = os.environ.get("MTNN_SPLIT_REG1024", "1")
for (m, n, k) in [(4096, 4096, 1024), (4096, 784, 1024), (1024, 1024, 1024), (16384, 16384, 1024), (2048, 8192, 1024), (128, 16384, 1024)]:
    wins, sp = [], []
    for rep in range(7):
        flush.sum(); torch.cuda._sleep(50000)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); e1.record()
        torch.cuda.synchronize()
        if rep: wins.append(e0.elapsed_time(e1) * 1e3)
        L.mtnn_profile_reset(); L.mtnn_profile_enable(1)
        flush.sum(); torch.cuda._sleep(50000)
        _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s))
        torch.cuda.synchronize(); L.mtnn_profile_enable(0)
        if rep: sp.append(_lib.profile_read(_lib.KCLASS_SPLIT)[0] * 1e3)
    print(f"reg1024={tag} nt ({m},{n},{k}) window {statistics.median(wins):7.1f} us split {statistics.median(sp):6.1f} us", flush=True)
