"""NN with k <= 16 (the FCN's 1024 x 4096 x 10 backward product): per-call time
and parity (event-timed after an L2 flush)."""
import os, statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device="cuda")
tag = os.environ.get("TAG", "")
for (m, n, k) in [(1024, 4096, 10), (4096, 4096, 10), (1024, 784, 10), (8192, 16384, 4), (1000, 1000, 16)]:
    a = torch.rand(m, k, device="cuda") * 2 - 1; bt = torch.rand(k, n, device="cuda") * 2 - 1
    c = torch.empty(m, n, device="cuda")
    _lib.check(L.mtnn_gemm_nn(a.data_ptr(), bt.data_ptr(), c.data_ptr(), m, n, k, 0, s))
    want = a.double() @ bt.double()
    err = ((c.double() - want).norm() / want.norm()).item()
    ev = []
    for rep in range(8):
        flush.sum(); torch.cuda._sleep(50000)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); _lib.check(L.mtnn_gemm_nn(a.data_ptr(), bt.data_ptr(), c.data_ptr(), m, n, k, 0, s)); e1.record()
        if rep >= 2: ev.append((e0, e1))
    torch.cuda.synchronize()
    t = statistics.median(x.elapsed_time(y) for x, y in ev) * 1e3
    print(f"{tag} nn ({m},{n},{k}) {t:7.1f} us {4.0 * m * n / t / 1e3:7.0f} GB/s (C writes) err {err:.2e}", flush=True)
