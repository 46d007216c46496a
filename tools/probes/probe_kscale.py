"""GEMM-only durations (run under ncu --metrics gpu__time_duration.sum) of one-wave
problems at growing k: t(k) = t0 + k * slope separates fixed per-tile cost from
the steady-state k-block rate. argv[1]: nt | pair."""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib, device
mode = sys.argv[1] if len(sys.argv) > 1 else "nt"
if mode == "pair":
    _lib.config_set("tc_pair", 2)
else:
    _lib.config_set("tc_pair", 0)
m, n = (1024, 4096) if mode != "pair" else (2048, 4096)
for k in (512, 1024, 2048, 4096, 8192, 16384):
    a = torch.rand(m, k, device="cuda"); b = torch.rand(n, k, device="cuda")
    for _ in range(3):
        device.gemm_nt(a, b, variant=3)
    torch.cuda.synchronize()
print("done")
