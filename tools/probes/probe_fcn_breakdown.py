"""FCN step (configs[3]) per call: window time (CUDA events around the call,
L2 flushed before) and per-kernel-class times of the same call (library
events on every launch), median of 5. python tools/probes/probe_fcn_breakdown.py"""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
widths = [784, 4096, 4096, 4096, 10]
layers = list(zip(widths[:-1], widths[1:]))
calls = [("nt", 1024, dout, din) for din, dout in layers]
for din, dout in reversed(layers):
    calls.append(("nn", 1024, din, dout)); calls.append(("nt", dout, din, 1024))
A = torch.rand(4096 * 4096, device=dev) * 2 - 1; B = torch.rand(4096 * 4096, device=dev) * 2 - 1
C = torch.empty(4096 * 4096, device=dev)
tot_w, tot_c = 0.0, {}
for (op, m, n, k) in calls:
    fn = L.mtnn_gemm_nt if op == "nt" else L.mtnn_gemm_nn
    wins, per = [], {c: [] for c in _lib.KCLASS_NAMES}
    for rep in range(6):
        flush.sum(); torch.cuda._sleep(100000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _lib.check(fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); b.record()
        torch.cuda.synchronize()
        if rep:
            wins.append(a.elapsed_time(b) * 1e3)
        L.mtnn_profile_reset(); L.mtnn_profile_enable(1)
        flush.sum(); torch.cuda._sleep(100000)
        _lib.check(fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s))
        torch.cuda.synchronize(); L.mtnn_profile_enable(0)
        if rep:
            for c in _lib.KCLASS_NAMES:
                ms, nl, _ = _lib.profile_read(c)
                if nl:
                    per[c].append(ms * 1e3)
    w = statistics.median(wins); tot_w += w
    parts = {_lib.KCLASS_NAMES[c]: statistics.median(v) for c, v in per.items() if v}
    for kk, v in parts.items():
        tot_c[kk] = tot_c.get(kk, 0) + v
    print(f"{op} ({m},{n},{k}) window {w:7.1f} us | " +
          " ".join(f"{kk} {v:6.1f}" for kk, v in parts.items()), flush=True)
print(f"total window {tot_w:.1f} us = {2.2614e11 / tot_w / 1e6:.1f} TF/s;", {k: round(v, 1) for k, v in tot_c.items()})
