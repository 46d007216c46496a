"""Small calls through every kernel family, for compute-sanitizer runs."""
import sys, numpy as np
sys.path.insert(0, ".")
import oracle
from paper_1702_03192_b200 import _lib, gemm_nt, gemm_nn, gemm_tnn, transpose_oop
rng = np.random.default_rng(5)
for (m, n, k) in [(128, 2048, 256), (2048, 128, 256), (300, 1100, 520), (256, 384, 264), (1024, 10, 512), (130, 260, 64)]:
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32); b = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    want = oracle.oracle_nt_blas(a, b)
    for v in ("auto", "tc3xf16s", "tc3xtf32", "ffma"):
        for fn in (gemm_nt, gemm_tnn):
            try:
                got = fn(a, b, variant=v)
            except Exception as e:
                print("skip", (m, n, k), v, fn.__name__, type(e).__name__); continue
            assert oracle.rel_frobenius(got, want) < 1e-5, ((m, n, k), v, fn.__name__)
    if n % 16 == 0:
        got = gemm_nn(a, np.ascontiguousarray(b.T))
        assert oracle.rel_frobenius(got, want) < 1e-5
    assert np.array_equal(transpose_oop(b), b.T)
# session-3 kernels: row split by k branch (reg / looped / CTA-register / smem),
# column split (strip / cluster / band), skinny NT
for (m, n, k) in [(384, 384, 256), (384, 384, 1024), (384, 384, 4104), (384, 384, 16392), (384, 384, 20000)]:
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32); b = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    assert oracle.rel_frobenius(gemm_nt(a, b, variant="tc3xf16s"), oracle.oracle_nt_blas(a, b)) < 1e-5
for (m, n, k) in [(384, 4096, 512), (384, 208, 1032), (384, 1072, 4104), (256, 384, 8200)]:
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32); bt = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    want = a.astype(np.float64) @ bt.astype(np.float64)
    assert oracle.rel_frobenius(gemm_nn(a, bt, variant="tc3xf16s"), want) < 1e-5
for (m, n, k) in [(1024, 10, 4096), (10, 4096, 1024), (300, 3, 64), (5, 7, 4)]:
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32); b = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    assert oracle.rel_frobenius(gemm_nt(a, b), oracle.oracle_nt_blas(a, b)) < 1e-5
# round 2: residual fix-up entries (outlier columns)
for (m, n, k) in [(256, 512, 1032), (384, 1024, 2048)]:
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32) * 1e-7; b = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    a[:, 3], b[:, 3] = 10.0, 0.0
    want = a.astype(np.float64) @ b.astype(np.float64).T
    assert oracle.rel_frobenius(gemm_nt(a, b, variant="tc3xf16s"), want) < 1e-5, (m, n, k)
# session 4: streaming skinny NT (clusters along k, second-pass fold, ragged)
for (m, n, k) in [(300, 10, 1024), (10, 300, 4100), (256, 10, 16384), (1, 1, 4), (77, 3, 2052)]:
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32); b = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    assert oracle.rel_frobenius(gemm_nt(a, b), oracle.oracle_nt_blas(a, b)) < 1e-5, (m, n, k)
print("sanitize run ok")
