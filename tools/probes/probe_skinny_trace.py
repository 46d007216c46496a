"""Per-CTA phase stamps of the tiled skinny kernel (trace build:
FILES=gemm_ffma.cu tools/build_variant.sh skinny_trace -DMTNN_TRACE)."""
import ctypes, os, sys, numpy as np, torch
os.environ.setdefault("MTNN_B200_LIB", "build/variants/skinny_trace/libmtnn_b200.so")
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device="cuda")
for (m, n, k) in [(1024, 10, 4096), (10, 4096, 1024)]:
    a = torch.rand(m, k, device="cuda"); b = torch.rand(n, k, device="cuda"); c = torch.empty(m, n, device="cuda")
    for rep in range(4):
        flush.sum(); torch.cuda._sleep(50000)
        _lib.check(L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, 0, s))
    torch.cuda.synchronize()
    buf = np.zeros(8192 * 8, dtype=np.uint64)
    _lib.check(L.mtnn_skinny_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(buf.size)))
    t = buf.reshape(-1, 8).astype(np.int64)
    t = t[t[:, 0] > 0]
    t = t[t[:, 0] > t[:, 0].max() - 10**8]  # this call's CTAs
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    print(f"({m},{n},{k}) per-phase us after the first CTA's entry: min / median / max")
    for p, name in enumerate(["entry", "pdl", "first loads", "chunk done", "-", "cluster bar1", "stores", "exit"]):
        col = rel[:, p]
        if name == "-": continue
        print(f"  {name:14s} {col.min():7.2f} {np.median(col):7.2f} {col.max():7.2f}")
