"""Floor for a 16 MB one-pass read at FCN GEMV size: torch copy / row-sum / our
skinny NT, event-timed after an L2 flush (per-call windows)."""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device="cuda")
a = torch.rand(1024, 4096, device="cuda"); b = torch.rand(10, 4096, device="cuda"); c = torch.empty(1024, 10, device="cuda")
d = torch.empty_like(a); r = torch.empty(1024, device="cuda")
def t(fn, n=10):
    ev = []
    for i in range(n):
        flush.sum(); torch.cuda._sleep(50000)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        if i >= 2: ev.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ev) * 1e3
print("copy 16MB        %.1f us" % t(lambda: d.copy_(a)))
print("rowsum 16MB      %.1f us" % t(lambda: torch.sum(a, dim=1, out=r)))
print("colsum 16MB      %.1f us" % t(lambda: torch.sum(a, dim=0)))
print("torch mv x10     %.1f us" % t(lambda: torch.mm(a, b.T, out=c)))
print("skinny nt        %.1f us" % t(lambda: _lib.check(L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), 1024, 10, 4096, 0, s))))
print("empty window     %.1f us" % t(lambda: None))
