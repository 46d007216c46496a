"""Per-call cost of the residual fix-up: back-to-back device NT calls with the
fix-up on / off (interleaved blocks), CUDA events around each block."""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import device, _lib, operands

shapes = [(128, 1024, 256), (256, 256, 4096), (1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096),
          (16384, 16384, 1024), (16384, 128, 16384), (128, 16384, 16384), (8192, 8192, 8192),
          (16384, 16384, 16384)]
for (m, n, k) in shapes:
    a, b = operands.make_operands(m, n, k, 0)  # the reference harness's operands
    c = torch.empty(m, n, device="cuda")
    reps = max(5, min(200, int(2e11 / (2 * m * n * k))))
    res = {0: [], 1: []}
    for rnd in range(6):
        for f in (0, 1):
            _lib.config_set("fixup", f)
            for _ in range(3):
                device.gemm_nt(a, b, out=c)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                device.gemm_nt(a, b, out=c)
            e1.record()
            torch.cuda.synchronize()
            res[f].append(e0.elapsed_time(e1) * 1e3 / reps)
    off, on = min(res[0]), min(res[1])
    print(f"{(m,n,k)}: off {off:.1f} us  on {on:.1f} us  delta {on-off:+.2f} us ({(on/off-1)*100:+.1f}%)", flush=True)
