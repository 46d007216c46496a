"""One FCN-shaped call for ncu: python tools/probes/fcn_one.py op m n k [reps]"""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import device
op, m, n, k = sys.argv[1], *map(int, sys.argv[2:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
torch.manual_seed(0)
a = torch.rand(m, k, device="cuda") * 2 - 1
b = torch.rand(n, k, device="cuda") * 2 - 1
bt = b.t().contiguous()
for _ in range(reps):
    device.gemm_nt(a, b) if op == "nt" else device.gemm_nn(a, bt)
torch.cuda.synchronize()
