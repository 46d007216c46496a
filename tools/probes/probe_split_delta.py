"""Per sweep case: operand-split and split-K-reduce kernel times with the
residual tracking on vs off (every launch event-timed), largest deltas."""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
s = [2 ** e for e in range(7, 15)]
A = torch.rand(16384 * 16384, device="cuda") * 2 - 1
B = torch.rand(16384 * 16384, device="cuda") * 2 - 1
C = torch.empty(16384 * 16384, device="cuda")
st = torch.cuda.current_stream().cuda_stream
cls = [_lib.KCLASS_SPLIT, _lib.KCLASS_REDUCE, _lib.KCLASS_FIXUP]
res = {}
L.mtnn_profile_enable(1)
for f in (0, 1):
    _lib.config_set("fixup", f)
    for m in s:
        for n in s:
            for k in s:
                _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, st))
                torch.cuda.synchronize()
                L.mtnn_profile_reset()
                for _ in range(3):
                    _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, st))
                torch.cuda.synchronize()
                res[(f, m, n, k)] = [_lib.profile_read(c)[0] * 1e3 / 3 for c in cls]
for ci, name in enumerate(("split", "reduce", "fixup")):
    tot0 = sum(v[ci] for key, v in res.items() if key[0] == 0)
    tot1 = sum(v[ci] for key, v in res.items() if key[0] == 1)
    print(f"{name}: off {tot0:.0f} us  on {tot1:.0f} us")
    d = sorted(((res[(1,) + key[1:]][ci] - v[ci], key[1:]) for key, v in res.items() if key[0] == 0), reverse=True)
    for x in d[:8]:
        print(f"    {x[0]:+8.1f} us {x[1]}  off {res[(0,)+x[1]][ci]:.1f}")
