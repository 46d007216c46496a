"""Where do rare slow FCN steps come from? The bench's timed loop (spin kernel,
event, call, event per call), 200 steps; for each call window: device time and
the host time spent enqueueing that call. A window far above its call's median
with a long host enqueue = a host stall counted as device idle time."""
import statistics, sys, time, ctypes, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
widths = [784, 4096, 4096, 4096, 10]
layers = list(zip(widths[:-1], widths[1:]))
calls = [("nt", 1024, dout, din) for din, dout in layers]
for din, dout in reversed(layers):
    calls.append(("nn", 1024, din, dout)); calls.append(("nt", dout, din, 1024))
A = torch.rand(4096 * 4096, device=dev); B = torch.rand(4096 * 4096, device=dev); C = torch.empty(4096 * 4096, device=dev)
rec = []
for st in range(200):
    ev = []
    for i, (op, m, n, k) in enumerate(calls):
        torch.cuda._sleep(200000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        a.record()
        fn = L.mtnn_gemm_nt if op == "nt" else L.mtnn_gemm_nn
        _lib.check(fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s))
        b.record()
        h1 = time.perf_counter()
        ev.append((i, a, b, (h1 - h0) * 1e6))
    torch.cuda.synchronize()
    for i, a, b, h in ev:
        rec.append((st, i, a.elapsed_time(b) * 1e3, h))
med = {i: statistics.median(r[2] for r in rec if r[1] == i) for i in range(len(calls))}
slow = [r for r in rec if r[2] > 1.5 * med[r[1]] + 5]
print(f"{len(rec)} windows, {len(slow)} slow (> 1.5x median + 5 us)")
for st, i, d, h in slow[:20]:
    print(f"  step {st} call {i}: device {d:.1f} us (median {med[i]:.1f}), host enqueue {h:.1f} us")
hs = sorted(r[3] for r in rec)
print("host enqueue us: median %.1f p99 %.1f max %.1f" % (hs[len(hs)//2], hs[int(len(hs)*0.99)], hs[-1]))
