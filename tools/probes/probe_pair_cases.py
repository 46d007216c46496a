"""Per-case interleaved A/B (tc_pair 0 vs 1) on the sweep cases that take the
pair kernel, median of 4 alternating reps."""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
A = torch.rand(16384 * 16384, device=dev) * 2 - 1; B = torch.rand(16384 * 16384, device=dev) * 2 - 1
C = torch.empty(16384 * 16384, device=dev)
E = [2 ** e for e in range(7, 15)]
rows = []
for m in E:
    for n in E:
        for k in E:
            if ((m + 255) // 256) * ((n + 255) // 256) < 74 or min(m, n) <= 256:
                continue
            ev = {0: [], 1: []}
            for rep in range(5):
                for mode in ((0, 1) if rep % 2 == 0 else (1, 0)):
                    _lib.config_set("tc_pair", mode)
                    flush.sum(); torch.cuda._sleep(200000)
                    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
                    a.record(); _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); b.record()
                    if rep: ev[mode].append((a, b))
            torch.cuda.synchronize()
            t0 = statistics.median(x.elapsed_time(y) for x, y in ev[0]); t1 = statistics.median(x.elapsed_time(y) for x, y in ev[1])
            rows.append((m, n, k, t0, t1))
print("cases", len(rows), "single %.1f ms pair %.1f ms" % (sum(r[3] for r in rows), sum(r[4] for r in rows)))
for r in rows:
    if r[4] > r[3] * 1.01 or r[3] > 1.0:
        print("(%d,%d,%d) single %.3f pair %.3f ratio %.3f" % (r[0], r[1], r[2], r[3], r[4], r[3] / r[4]))
