"""One tensor-core call for compute-sanitizer racecheck: python tools/probes/race_one.py m n k [nn]"""
import sys, numpy as np
sys.path.insert(0, ".")
from paper_1702_03192_b200 import gemm_nt, gemm_nn
m, n, k = map(int, sys.argv[1:4])
rng = np.random.default_rng(1)
a = rng.uniform(-1, 1, (m, k)).astype(np.float32); b = rng.uniform(-1, 1, (n, k)).astype(np.float32)
if len(sys.argv) > 4:
    gemm_nn(a, np.ascontiguousarray(b.T), variant="tc3xf16s")
else:
    gemm_nt(a, b, variant="tc3xf16s")
print("ok")
