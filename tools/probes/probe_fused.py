"""Interleaved A/B of the fused operand split (knob fused_split 0 vs 2) per NT
shape: whole calls (split + GEMM + fix-up), median of reps, best of rounds."""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
A = torch.rand(16384 * 16384, device=dev) * 2 - 1; B = torch.rand(16384 * 16384, device=dev) * 2 - 1
C = torch.empty(16384 * 16384, device=dev)


def t_case(m, n, k, mode, reps=5):
    _lib.config_set("fused_split", mode)
    ev = []
    for rep in range(reps + 1):
        flush.sum(); torch.cuda._sleep(200000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 3, s)); b.record()
        if rep: ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


shapes = [(1024, 4096, 784), (1024, 4096, 4096), (4096, 4096, 1024), (4096, 784, 1024), (1024, 1024, 16384),
          (2048, 2048, 4096), (512, 4096, 4096), (2048, 2048, 2048), (1024, 2048, 8192), (4096, 1024, 4096),
          (256, 8192, 4096)]
for m, n, k in shapes:
    r = {}
    for rep in range(3):
        for mode in (0, 2):
            r.setdefault(mode, []).append(t_case(m, n, k, mode, reps=3))
    t0, t2 = min(r[0]) * 1e3, min(r[2]) * 1e3
    f = 2 * m * n * k / 1e9
    print(f"nt ({m},{n},{k}) presplit {t0:.1f} us {f/t0:.0f} TF/s | fused {t2:.1f} us {f/t2:.0f} TF/s | {t0/t2:.3f}x", flush=True)
