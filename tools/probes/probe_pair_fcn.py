"""Interleaved A/B of CTA-pair tiles (tc_pair 2 = forced) vs the default rule on
the FCN step's tensor-core calls (whole calls, median of reps, best of rounds)."""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
A = torch.rand(8192 * 8192, device=dev) * 2 - 1; B = torch.rand(8192 * 8192, device=dev) * 2 - 1
C = torch.empty(8192 * 8192, device=dev)
def t_case(op, m, n, k, mode, reps=5):
    _lib.config_set("tc_pair", mode)
    fn = L.mtnn_gemm_nt if op == "nt" else L.mtnn_gemm_nn
    ev = []
    for rep in range(reps + 1):
        flush.sum(); torch.cuda._sleep(200000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _lib.check(fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 3, s)); b.record()
        if rep: ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)
shapes = [("nt", 1024, 4096, 784), ("nt", 1024, 4096, 4096), ("nn", 1024, 4096, 4096), ("nn", 1024, 784, 4096),
          ("nt", 4096, 784, 1024), ("nt", 4096, 4096, 1024), ("nt", 512, 4096, 4096), ("nt", 2048, 2048, 2048),
          ("nt", 1024, 2048, 4096), ("nt", 2048, 2048, 8192), ("nt", 1024, 8192, 1024), ("nt", 2048, 4096, 1024)]
for op, m, n, k in shapes:
    r = {}
    for rep in range(3):
        for mode in (1, 2):
            r.setdefault(mode, []).append(t_case(op, m, n, k, mode, reps=3))
    t1, t2 = min(r[1]) * 1e3, min(r[2]) * 1e3
    print(f"{op} ({m},{n},{k}) default {t1:.1f} us | pairs {t2:.1f} us | {t1/t2:.3f}x", flush=True)
