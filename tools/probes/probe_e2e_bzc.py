"""Interleaved per-case A/B at k > 4096: B-first pipeline vs the blocked
pipeline with SM-store C blocks (run with MTNN_PIPE_BLOCKED_MAXK=16384)."""
import os, sys, time, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
E = [2 ** e for e in range(7, 15)]
KS = [int(x) for x in os.environ.get("KS", "8192,16384").split(",") if x]
shapes = [(m, n, k) for m in E for n in E for k in KS if n >= 1024 and 4 * (m * k + n * k + m * n) >= 8 << 20]
ha = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hb = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hc = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory()
tot = {0: 0.0, 1: 0.0}
for (m, n, k) in shapes:
    ts = {0: [], 1: []}
    for rep in range(3):
        for v in (0, 1):
            _lib.config_set("host_pipeline_blocked", v)
            _lib.config_set("host_pipeline_zc", v)
            t0 = time.perf_counter()
            _lib.check(L.mtnn_gemm_nt_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, 0))
            ts[v].append(time.perf_counter() - t0)
    med = {v: sorted(ts[v])[1] for v in (0, 1)}
    for v in (0, 1): tot[v] += med[v]
    print(f"{m} {n} {k} bfirst {med[0]*1e3:.3f} blockedzc {med[1]*1e3:.3f}", flush=True)
print("total B-first %.1f ms, blocked+zc %.1f ms" % (tot[0] * 1e3, tot[1] * 1e3))
