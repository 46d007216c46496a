"""In-kernel F16S split shapes (short side <= 256): per-call device time, for
A/B of the h/l and raw ring depths (build variants via MTNN_B200_LIB)."""
import os, statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device="cuda")
A = torch.rand(16384 * 16384, device="cuda"); B = torch.rand(16384 * 16384, device="cuda"); C = torch.empty(16384 * 16384, device="cuda")
tag = os.environ.get("TAG", "")
tot = 0.0
for (m, n, k) in [(128, 16384, 16384), (16384, 128, 16384), (256, 16384, 8192), (16384, 256, 4096), (128, 4096, 4096),
                  (256, 2048, 2048), (2048, 128, 16384), (128, 8192, 1024)]:
    wins = []
    for rep in range(7):
        flush.sum(); torch.cuda._sleep(50000)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); e1.record()
        if rep: wins.append((e0, e1))
    torch.cuda.synchronize()
    t = statistics.median(x.elapsed_time(y) for x, y in wins) * 1e3
    tot += t
    print(f"{tag} nt ({m},{n},{k}) {t:8.1f} us", flush=True)
print(f"{tag} total {tot:.1f} us")
