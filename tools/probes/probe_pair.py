import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_1702_03192_b200 import _lib, gemm_nt
rng = np.random.default_rng(1)
for (m, n, k) in [(256, 256, 64), (512, 768, 320), (300, 520, 136), (2560, 2048, 1024)]:
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32); b = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    want = oracle.oracle_nt_blas(a, b)
    for v in ("tc3xf16s", "tc3xtf32"):
        _lib.config_set("tc_pair", 0); ref = gemm_nt(ta, tb, variant=v).cpu().numpy()
        _lib.config_set("tc_pair", 2); got = gemm_nt(ta, tb, variant=v).cpu().numpy()
        torch.cuda.synchronize()
        print((m, n, k), v, "pair err %.2e single err %.2e identical %s" % (
            oracle.rel_frobenius(got, want), oracle.rel_frobenius(ref, want), np.array_equal(got, ref)), flush=True)
