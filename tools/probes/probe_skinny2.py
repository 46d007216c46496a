"""Skinny-shape breakdown: per variant, median time and per-kernel-class ms.
Run twice (MTNN_TF32_INKERNEL=0/1) — the env is read once per process."""
import os, sys, statistics, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
shapes = [(128, 16384, 16384), (16384, 128, 16384), (256, 16384, 16384), (512, 16384, 16384),
          (1024, 16384, 16384), (8192, 128, 16384), (16384, 1024, 16384), (128, 8192, 8192),
          (16384, 16384, 256), (16384, 16384, 512), (2048, 2048, 2048), (8192, 8192, 8192)]
tag = os.environ.get("MTNN_TF32_INKERNEL", "0")
A = torch.rand(16384 * 16384, device=dev) * 2 - 1
B = torch.rand(16384 * 16384, device=dev) * 2 - 1
C = torch.empty(16384 * 16384, device=dev)
for (m, n, k) in shapes:
    out = []
    for v in (3, 1):
        f = lambda: _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, v, s))
        f(); f()
        L.mtnn_profile_reset(); L.mtnn_profile_enable(1)
        ev = []
        for _ in range(5):
            flush.sum(); torch.cuda._sleep(200000)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); ev.append((a, b))
        torch.cuda.synchronize()
        L.mtnn_profile_enable(0)
        t = statistics.median(a.elapsed_time(b) for a, b in ev)
        prof = {_lib.KCLASS_NAMES[c]: _lib.profile_read(c)[0] / 5 for c in _lib.KCLASS_NAMES}
        br = " ".join(f"{k[:6]}={v:.3f}" for k, v in prof.items() if v > 0)
        out.append(f"{'f16s' if v == 3 else 'tf32'}:{t:.3f}ms {2*m*n*k/t/1e9:.0f}TF [{br}]")
    print(f"inkernel={tag} ({m},{n},{k}) " + " | ".join(out), flush=True)
