"""Intra-row dynamic range probe: rel-Frobenius (whole C and worst row) of every
variant on adversarial inputs vs float64."""
import numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_1702_03192_b200 import device, _lib

def cases(rng, m, n, k):
    U = lambda *s: rng.uniform(-1, 1, s)
    a = U(m, k) * 1e-7; a[:, 0] = 1; b = U(n, k); b[:, 0] = 0
    yield "outlier1e7_masked", a, b
    a = np.full((m, k), 1e-6); a[:, 0] = 1e6; b = np.ones((n, k)); b[:, 0] = 0
    yield "outlier1e12_const", a, b
    a = U(m, k); a[:, 3] *= 1e8; b = U(n, k); b[:, 3] = 0
    yield "col3x1e8_masked", a, b
    a = U(m, k); a[:, 3] *= 1e8; b = U(n, k)
    yield "col3x1e8_unmasked", a, b
    a = U(m, k); b = U(n, k); b[:, 5] *= 1e9; a[:, 5] = 0
    yield "Bcol5x1e9_masked", a, b
    a = U(m, k) * 1e-41; b = U(n, k) * 1e30
    yield "A_subnormal", a, b
    a = U(m, k) * 10.0 ** rng.uniform(-12, 12, (m, k)); b = U(n, k) * 10.0 ** rng.uniform(-6, 6, (n, k))
    yield "mixed_1e12", a, b
    a = U(m, k); b = U(n, k)
    yield "uniform", a, b

def err(got, want):
    d = got.astype(np.float64) - want
    fro = np.linalg.norm(d) / max(np.linalg.norm(want), 1e-300)
    rows = np.linalg.norm(d, axis=1) / np.maximum(np.linalg.norm(want, axis=1), 1e-300)
    return fro, rows.max()

rng = np.random.default_rng(0)
for (m, n, k) in [(512, 512, 4096), (256, 2048, 1024), (2048, 128, 2048)]:
    for name, a, b in cases(rng, m, n, k):
        a32 = a.astype(np.float32); b32 = b.astype(np.float32)
        want = a32.astype(np.float64) @ b32.astype(np.float64).T
        ta = torch.from_numpy(a32).cuda(); tb = torch.from_numpy(b32).cuda()
        line = []
        for vn in ("auto", "tc3xf16s", "tc3xtf32", "ffma"):
            v = _lib.VARIANTS[vn]
            for path, fn in (("nt", device.gemm_nt), ("tnn", device.gemm_tnn)):
                try:
                    got = fn(ta, tb, variant=v).cpu().numpy()
                    f, r = err(got, want)
                    line.append(f"{vn}/{path} {f:.1e}/{r:.1e}" + (" FAIL" if r > 1e-5 else ""))
                except Exception as e:
                    line.append(f"{vn}/{path} ERR {e}")
        print(f"({m},{n},{k}) {name}: " + " | ".join(line), flush=True)
