"""Runs one NT shape a few times (for ncu): python one_case.py m n k [fixup]"""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import device, _lib
m, n, k = map(int, sys.argv[1:4])
if len(sys.argv) > 4:
    _lib.config_set("fixup", int(sys.argv[4]))
a = torch.rand(m, k, device="cuda") * 2 - 1
b = torch.rand(n, k, device="cuda") * 2 - 1
c = torch.empty(m, n, device="cuda")
for _ in range(3):
    device.gemm_nt(a, b, out=c)
torch.cuda.synchronize()
