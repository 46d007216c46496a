"""Interleaved A/B of the f16s in-kernel split threshold on the sweep cases it
affects: per case, thresholds alternate within each rep (median of 5)."""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
E = [2 ** e for e in range(7, 15)]
knobs = [int(x) for x in sys.argv[1:]] or [0, 128, 256, 512]
shapes = [(m, n, k) for m in E for n in E for k in E if min(m, n) <= max(knobs) and max(m, n) >= 1024]
A = torch.rand(16384 * 16384, device=dev) * 2 - 1
B = torch.rand(16384 * 16384, device=dev) * 2 - 1
C = torch.empty(16384 * 16384, device=dev)
tot = {t: 0.0 for t in knobs}
by_short = {}
for (m, n, k) in shapes:
    ev = {t: [] for t in knobs}
    for rep in range(6):
        for t in knobs:
            _lib.config_set("f16s_inkernel_max_short", t)
            flush.sum(); torch.cuda._sleep(200000)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); b.record()
            if rep: ev[t].append((a, b))
    torch.cuda.synchronize()
    med = {t: statistics.median(a.elapsed_time(b) for a, b in ev[t]) for t in knobs}
    for t in knobs:
        tot[t] += med[t]
        by_short.setdefault(min(m, n), {}).setdefault(t, 0.0)
        by_short[min(m, n)][t] += med[t]
print("cases", len(shapes), "totals ms", {t: round(v, 2) for t, v in tot.items()})
for sh in sorted(by_short):
    print("short side", sh, {t: round(v, 2) for t, v in by_short[sh].items()})
