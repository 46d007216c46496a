"""FCN step (configs[3] call list) repeated with per-call event windows, as
bench.py times it, under tc_streamk 0 and 1: per-step totals and the slowest
windows (looks for outliers)."""
import sys, torch
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
for mode in (0, 1, 0, 1):
    _lib.config_set("tc_streamk", mode)
    steps = []
    for st in range(25):
        ev = []
        for op, m, n, k in calls:
            torch.cuda._sleep(50000)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            fn = L.mtnn_gemm_nt if op == "nt" else L.mtnn_gemm_nn
            a.record(); _lib.check(fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); b.record()
            ev.append((a, b))
        torch.cuda.synchronize()
        steps.append([a.elapsed_time(b) * 1e3 for a, b in ev])
    tot = sorted(sum(x) for x in steps)
    worst = max((max(x), x.index(max(x))) for x in steps)
    print(f"sk={mode} step us: min {tot[0]:.0f} med {tot[len(tot)//2]:.0f} max {tot[-1]:.0f}; worst window {worst[0]:.0f} us (call {worst[1]})", flush=True)
