import sys, numpy as np
sys.path.insert(0, ".")
import oracle
from paper_1702_03192_b200 import gemm_nt, _lib
rng = np.random.default_rng(0)
for (m, n, k) in [(1, 1, 65536), (4, 4, 65536), (1, 1, 4096), (1, 4, 65536), (4, 1, 65536), (128, 128, 65536), (1, 1, 16384), (1, 8, 32768)]:
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32); b = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    want = oracle.oracle_nt_blas(a, b)
    out = []
    for v in ("tc3xf16s", "tc3xtf32", "ffma"):
        try:
            got = gemm_nt(a, b, variant=v)
            out.append(f"{v} {oracle.rel_frobenius(got, want):.1e} nan={np.isnan(got).sum()}")
        except Exception as e:
            out.append(f"{v} ERR {type(e).__name__}")
    print((m, n, k), " | ".join(out), flush=True)
