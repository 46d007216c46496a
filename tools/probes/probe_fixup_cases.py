"""Fix-up kernel time per sweep case (class 6 timed alone), top cases."""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import device, _lib
L = _lib.lib
s = [2 ** e for e in range(7, 15)]
A = torch.rand(16384 * 16384, device="cuda") * 2 - 1
B = torch.rand(16384 * 16384, device="cuda") * 2 - 1
C = torch.empty(16384 * 16384, device="cuda")
st = torch.cuda.current_stream().cuda_stream
rows = []
L.mtnn_profile_enable_classes(1 << _lib.KCLASS_FIXUP)
for m in s:
    for n in s:
        for k in s:
            _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, st))
            torch.cuda.synchronize()
            L.mtnn_profile_reset()
            _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, st))
            torch.cuda.synchronize()
            ms, nl, w = _lib.profile_read(_lib.KCLASS_FIXUP)
            rows.append((ms * 1e3, m, n, k))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(f"total fixup us over sweep: {tot:.0f}; median {sorted(r[0] for r in rows)[len(rows)//2]:.1f}")
for r in rows[:25]:
    print(f"{r[0]:8.1f} us  {r[1:]}")
