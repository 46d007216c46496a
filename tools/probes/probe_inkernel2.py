import sys, numpy as np
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib, gemm_nt
np.set_printoptions(linewidth=200, precision=3, suppress=True)
m, n, k = 128, 1024, 32
A = np.ones((m, k), np.float32)
for name, B in [("ones", np.ones((n, k), np.float32)),
                ("row=j", np.repeat(np.arange(n, dtype=np.float32)[:, None] / 1024, k, 1)),
                ("col=kk", np.repeat(np.arange(k, dtype=np.float32)[None, :] / 32, n, 0))]:
    B = np.ascontiguousarray(B)
    _lib.config_set("f16s_inkernel_max_short", 0); pre = gemm_nt(A, B, variant="tc3xf16s")
    _lib.config_set("f16s_inkernel_max_short", 1 << 20); ink = gemm_nt(A, B, variant="tc3xf16s")
    print(name, "pre row0[:8]", pre[0, :8], "ink row0[:8]", ink[0, :8])
    print("   ink rows 0..3 cols 0..8:\n", ink[:4, :9], "\n   ink col0 rows", ink[:16, 0])
# A converted (n small)
A2 = np.repeat(np.arange(1024, dtype=np.float32)[:, None] / 1024, 32, 1); B2 = np.ones((128, 32), np.float32)
_lib.config_set("f16s_inkernel_max_short", 1 << 20); ink = gemm_nt(np.ascontiguousarray(A2), B2, variant="tc3xf16s")
print("conv1 col0 rows[:12]", ink[:12, 0], "want", (np.arange(12) / 1024 * 32))
