"""One library call on cuda:0 for ncu captures: python tools/one_call.py nt|nn m n k [reps] [variant]."""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
op, m, n, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
variant = int(sys.argv[6]) if len(sys.argv) > 6 else 3
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
A = torch.rand(m * k, device=dev); B = torch.rand(n * k, device=dev); C = torch.empty(m * n, device=dev)
fn = L.mtnn_gemm_nt if op == "nt" else L.mtnn_gemm_nn
for _ in range(reps):
    _lib.check(fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, variant, s))
torch.cuda.synchronize()
