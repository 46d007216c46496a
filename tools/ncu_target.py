"""Small driver for ncu --set full captures of the hot kernels (one launch each)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import device

which = sys.argv[1] if len(sys.argv) > 1 else "nt8192"
VARIANT = int(sys.argv[2]) if len(sys.argv) > 2 else 3  # 3 = tc3xf16s, 1 = tc3xtf32
torch.manual_seed(0)
cases = {"nt8192": ("nt", 8192, 8192, 8192), "nt16384": ("nt", 16384, 16384, 16384),
         "nn16384": ("nn", 16384, 16384, 16384), "tr16384": ("tr", 16384, 16384, 0),
         "nt4096": ("nt", 4096, 4096, 4096), "skinny_m128": ("nt", 128, 16384, 16384),
         "skinny_n128": ("nt", 16384, 128, 16384), "skinny_m256": ("nt", 256, 16384, 16384),
         "smallk256": ("nt", 16384, 16384, 256), "nn1024x4096x4096": ("nn", 1024, 4096, 4096),
         "fcn10": ("nt", 1024, 10, 4096), "nt1024x4096x4096": ("nt", 1024, 4096, 4096),
         "nt4096x4096x1024": ("nt", 4096, 4096, 1024)}
op, m, n, k = cases[which]
if op == "tr":
    b = torch.rand(m, n, device="cuda"); out = torch.empty(n, m, device="cuda")
    for _ in range(3):
        device.transpose(b, out=out)
else:
    a = torch.rand(m, k, device="cuda"); b = torch.rand(n, k, device="cuda")
    bt = b.t().contiguous()
    for _ in range(2):
        if op == "nt":
            device.gemm_nt(a, b, variant=VARIANT)
        else:
            device.gemm_nn(a, bt, variant=VARIANT)
torch.cuda.synchronize()
print("done", which)
