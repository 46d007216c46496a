"""FCN step through the host-buffer C-ABI, per call: wall time vs the per-call
PCIe floor max(H2D / 55.5, D2H / 54.2, (H2D + D2H) / 93 GB/s)."""
import ctypes, sys, time, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
import os
L = _lib.lib
if os.environ.get("ZC"):
    _lib.config_set("host_pipeline_zc", int(os.environ["ZC"]))
if os.environ.get("BLOCKED"):
    _lib.config_set("host_pipeline_blocked", int(os.environ["BLOCKED"]))
widths = [784, 4096, 4096, 4096, 10]
layers = list(zip(widths[:-1], widths[1:]))
calls = [("nt", 1024, dout, din) for din, dout in layers]
for din, dout in reversed(layers):
    calls.append(("nn", 1024, din, dout)); calls.append(("grad", dout, din, 1024))
ha = torch.empty(4096 * 4096, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hb = torch.empty(4096 * 4096, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hc = torch.empty(4096 * 4096, dtype=torch.float32).pin_memory()
handle = ctypes.c_void_p()
prefix = _lib.default_prefix() if hasattr(_lib, "default_prefix") else None
T = F = 0.0
for (op, m, n, k) in calls:
    ts = []
    for rep in range(5):
        t0 = time.perf_counter()
        if op == "nn":
            rc = L.mtnn_gemm_nn_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, 0)
        else:
            rc = L.mtnn_gemm_nt_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, 0)
        _lib.check(rc)
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[2]
    h2d, d2h = 4 * (m * k + n * k), 4 * m * n
    floor = max(h2d / 55.5e9, d2h / 54.2e9, (h2d + d2h) / 93e9)
    T += t; F += floor
    print(f"{op:4s} ({m},{n},{k}) {t*1e3:7.3f} ms floor {floor*1e3:6.3f} ms  in {h2d/1e6:5.1f} MB out {d2h/1e6:5.1f} MB", flush=True)
print(f"step {T*1e3:.2f} ms, per-call floor {F*1e3:.2f} ms")
