"""Long randomized parity run (not part of the suite): random shapes x entry
points x variants x knob settings against the float64 oracle."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_1702_03192_b200 import _lib, gemm_nt, gemm_nn, gemm_tnn
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
N = int(sys.argv[2]) if len(sys.argv) > 2 else 200
rng = np.random.default_rng(seed)
picks = [1, 2, 3, 4, 7, 8, 9, 16, 31, 32, 33, 64, 96, 127, 128, 129, 192, 255, 256, 257, 384, 500, 512,
         513, 768, 1000, 1023, 1024, 1025, 1536, 2047, 2048, 2049, 3000, 4100]
bad = 0
longk = [4104, 6000, 8192, 8200, 12000, 16384, 16392, 20000]
import os
big = os.environ.get("FUZZ_BIG") == "1"
skinny = os.environ.get("FUZZ_SKINNY") == "1"  # GEMV-class: one output side 1..16
for it in range(N):
    m, n, k = (int(rng.choice(picks)) if rng.random() < 0.7 else int(rng.integers(1, 4200)) for _ in range(3))
    if it % 4 == 3:  # long-k branches of the row / column splits (register, cluster, band, smem)
        m, n, k = int(rng.choice(picks[:24])), int(rng.choice(picks[:24])), int(rng.choice(longk))
    if big and it % 4 == 1:  # one large output side: CTA pairs, grouped raster, split-K edges
        dims = [int(rng.choice([4096, 6000, 8192, 10000, 16384])), int(rng.choice(picks)),
                int(rng.choice([256, 1000, 2048, 4104]))]
        m, n, k = (dims[0], dims[1], dims[2]) if rng.random() < 0.5 else (dims[1], dims[0], dims[2])
    if skinny and it % 2 == 0:  # register / staged / streaming skinny kernels, clusters along k
        sm = int(rng.integers(1, 17))
        lg = int(rng.choice([1, 33, 300, 1024, 4096, 9000]))
        k = int(rng.choice([4, 64, 1028, 2052, 4096, 8192, 16384, 20000])) if rng.random() < 0.8 else int(rng.integers(1, 9000))
        m, n = (sm, lg) if rng.random() < 0.5 else (lg, sm)
    knobs = {"tc_pair": int(rng.integers(0, 3)), "f16s_inkernel_max_short": int(rng.choice([0, 256, 1 << 20])),
             "host_pipeline_blocked": int(rng.integers(0, 2))}
    for kk, vv in knobs.items():
        _lib.config_set(kk, vv)
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32); b = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    rows = np.unique(rng.choice(m, min(m, 16), replace=False))
    want = oracle.oracle_nt_rows(a, b, rows, np.arange(n))
    res = {}
    for v in ("auto", "tc3xf16s", "tc3xtf32", "ffma"):
        try:
            res["nt/" + v] = gemm_nt(a, b, variant=v)
        except RuntimeError:
            pass
    res["tnn"] = gemm_tnn(a, b)
    res["nn"] = gemm_nn(a, np.ascontiguousarray(b.T))
    res["dev"] = gemm_nt(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    for name, got in res.items():
        e = oracle.rel_frobenius(got[rows], want) if want.size and np.abs(want).sum() > 0 else 0.0
        if not (e < 1e-5):
            bad += 1
            print("FAIL", (m, n, k), knobs, name, e, flush=True)
print(f"seed {seed}: {N} shapes, {bad} failures", flush=True)
