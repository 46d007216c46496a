"""Per-class kernel times (every launch event-timed) for given shapes, fix-up on/off."""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import device, _lib
L = _lib.lib
shapes = [tuple(map(int, s.split("x"))) for s in (sys.argv[1:] or ["1024x1024x1024", "128x1024x256"])]
for (m, n, k) in shapes:
    a = torch.rand(m, k, device="cuda") * 2 - 1
    b = torch.rand(n, k, device="cuda") * 2 - 1
    c = torch.empty(m, n, device="cuda")
    for f in (0, 1):
        _lib.config_set("fixup", f)
        for _ in range(3):
            device.gemm_nt(a, b, out=c)
        torch.cuda.synchronize()
        L.mtnn_profile_enable(1)
        L.mtnn_profile_reset()
        for _ in range(20):
            device.gemm_nt(a, b, out=c)
        torch.cuda.synchronize()
        out = {}
        for kc, name in _lib.KCLASS_NAMES.items():
            ms, nl, w = _lib.profile_read(kc)
            if nl:
                out[name] = f"{ms * 1e3 / 20:.1f}us x{nl // 20}"
        L.mtnn_profile_enable(0)
        print((m, n, k), "fixup", f, out, flush=True)
