"""Interleaved A/B of the blocked host pipeline's C-block D2H: copy-engine 2-D
copies vs SM stores into the mapped host C (host_pipeline_zc), per case, over the
sweep's blocked-path cases (KS=... selects k; MAXK lifts the k <= 4096 gate)."""
import os, sys, time, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
E = [2 ** e for e in range(7, 15)]
KS = [int(x) for x in os.environ.get("KS", "").split(",") if x] or E
shapes = [(m, n, k) for m in E for n in E for k in KS if n >= 1024 and 4 * (m * k + n * k + m * n) >= 8 << 20]
ha = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hb = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hc = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory()
tot = {0: 0.0, 1: 0.0}
rows = []
for (m, n, k) in shapes:
    ts = {0: [], 1: []}
    for rep in range(3):
        for v in (0, 1):
            _lib.config_set("host_pipeline_zc", v)
            t0 = time.perf_counter()
            _lib.check(L.mtnn_gemm_nt_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, 0))
            ts[v].append(time.perf_counter() - t0)
    med = {v: sorted(ts[v])[1] for v in (0, 1)}
    for v in (0, 1): tot[v] += med[v]
    rows.append((med[1] - med[0], (m, n, k), med[0] * 1e3, med[1] * 1e3))
print("cases", len(shapes), "copy engine %.1f ms, SM stores %.1f ms" % (tot[0] * 1e3, tot[1] * 1e3))
rows.sort()
for w in rows[:6] + rows[-6:]: print(w[1], "CE %.2f SM %.2f" % (w[2], w[3]))
