import sys, numpy as np
sys.path.insert(0, ".")
import oracle
from paper_1702_03192_b200 import _lib, gemm_nt
rng = np.random.default_rng(0)
for (m, n, k) in [(128, 4096, 2048), (4096, 128, 2048), (128, 1024, 32), (128, 1024, 64), (128, 1024, 256)]:
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32); b = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    want = oracle.oracle_nt_blas(a, b)
    _lib.config_set("f16s_inkernel_max_short", 0); pre = gemm_nt(a, b, variant="tc3xf16s")
    _lib.config_set("f16s_inkernel_max_short", 1 << 20); ink = gemm_nt(a, b, variant="tc3xf16s")
    d = pre != ink
    print((m, n, k), "err pre %.2e ink %.2e" % (oracle.rel_frobenius(pre, want), oracle.rel_frobenius(ink, want)),
          "nan", np.isnan(ink).sum(), "diff frac %.3f" % d.mean(), "rows", np.unique(np.nonzero(d)[0])[:8], "cols", np.unique(np.nonzero(d)[1])[:8])
    if d.any():
        i, j = np.argwhere(d)[0]; print("  sample", pre[i, j], ink[i, j], want[i, j])
