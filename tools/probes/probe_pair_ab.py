"""Interleaved A/B: CTA-pair tiles vs single-CTA tiles (knob tc_pair), per shape,
plus the whole sweep total under each setting (interleaved per case)."""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
A = torch.rand(16384 * 16384, device=dev) * 2 - 1; B = torch.rand(16384 * 16384, device=dev) * 2 - 1
C = torch.empty(16384 * 16384, device=dev)
def t_case(m, n, k, mode, reps=5):
    ev = []
    _lib.config_set("tc_pair", mode)
    for rep in range(reps + 1):
        flush.sum(); torch.cuda._sleep(200000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); b.record()
        if rep: ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
for (m, n, k) in [(4096, 4096, 4096), (8192, 8192, 8192), (16384, 16384, 16384), (16384, 4096, 16384),
                  (2048, 16384, 16384), (16384, 16384, 1024), (4096, 4096, 16384)]:
    r = {}
    for rep in range(2):
        for mode in (0, 1):
            r.setdefault(mode, []).append(t_case(m, n, k, mode, reps=3))
    t0, t1 = min(r[0]), min(r[1])
    print(f"({m},{n},{k}) single {t0:.3f} ms {2*m*n*k/t0/1e9:.0f} TF/s | pair {t1:.3f} ms {2*m*n*k/t1/1e9:.0f} TF/s | {t0/t1:.3f}x", flush=True)
E = [2 ** e for e in range(7, 15)]
tot = {0: 0.0, 1: 0.0}
for m in E:
    for n in E:
        for k in E:
            for mode in (0, 1):
                tot[mode] += t_case(m, n, k, mode, reps=2)
F = 2 * 32640 ** 3
print("sweep single %.1f ms (%.0f TF/s)  pair %.1f ms (%.0f TF/s)" % (tot[0], F / tot[0] / 1e9, tot[1], F / tot[1] / 1e9))
