"""Host-buffer NT time per case under the blocked pipeline's k cap (env
MTNN_PIPE_BLOCKED_MAXK is read once per process, so each setting runs in its
own process: argv[1] = cap); prints per-case ms for the large-k cases."""
import sys, time, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
ha = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hb = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hc = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory()
cases = [(m, n, k) for k in (8192, 16384) for m in (2048, 4096, 8192, 16384) for n in (4096, 8192, 16384)]
tot = 0.0
out = []
for (m, n, k) in cases:
    ts = []
    for rep in range(4):
        t0 = time.perf_counter()
        _lib.check(L.mtnn_gemm_nt_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, 0))
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[1]
    tot += t
    out.append(f"{m}x{n}x{k}:{t*1e3:.2f}")
print(sys.argv[1], f"total {tot*1e3:.1f} ms |", " ".join(out), flush=True)
