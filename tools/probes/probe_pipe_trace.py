"""Timeline of the blocked host pipeline (MTNN_PIPE_TRACE=1): one call per shape
after a warm-up, wall time printed; spans go to stderr."""
import os, sys, time, torch
os.environ["MTNN_PIPE_TRACE"] = "1"
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
shapes = [tuple(map(int, x.split("x"))) for x in (sys.argv[1:] or ["8192x16384x4096"])]
mx = max(max(m * k, n * k, m * n) for m, n, k in shapes)
ha = torch.empty(mx, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hb = torch.empty(mx, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hc = torch.empty(mx, dtype=torch.float32).pin_memory()
for (m, n, k) in shapes:
    _lib.check(L.mtnn_gemm_nt_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, 0))
    sys.stderr.flush()
    print(f"== {m}x{n}x{k}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    _lib.check(L.mtnn_gemm_nt_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, 0))
    print(f"== {m}x{n}x{k} wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
