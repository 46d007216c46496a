"""GEMV-class NT products (output side <= 16): parity against fp64 and per-call
device time, for the A/B of MTNN_SKINNY_TILE / MTNN_SKINNY_STAGED."""
import os, statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device="cuda")
tag = os.environ.get("TAG", "")
for (m, n, k) in [(1024, 10, 4096), (10, 4096, 1024), (4096, 10, 1024), (1024, 16, 4096), (1024, 4, 4096),
                  (8192, 8, 8192), (1, 4096, 4096), (16, 65536, 512), (100000, 10, 784), (777, 13, 1028),
                  (33, 3, 6000), (2048, 10, 16384)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.rand(m, k, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, k, device="cuda", generator=g) * 2 - 1
    c = torch.empty(m, n, device="cuda")
    _lib.check(L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, 0, s))
    want = a.double() @ b.double().T
    err = ((c.double() - want).norm() / want.norm()).item()
    ev = []
    for rep in range(8):
        flush.sum(); torch.cuda._sleep(50000)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); _lib.check(L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, 0, s)); e1.record()
        if rep >= 2: ev.append((e0, e1))
    torch.cuda.synchronize()
    t = statistics.median(x.elapsed_time(y) for x, y in ev) * 1e3
    gbs = 4.0 * (m * k + n * k + m * n) / t / 1e3
    print(f"{tag} nt ({m},{n},{k}) {t:7.1f} us {gbs:7.0f} GB/s err {err:.2e}", flush=True)
