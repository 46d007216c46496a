"""The FCN's three GEMV-class products, one call each (run under ncu for
kernel-only durations): NT 1024x10x4096, NN 1024x4096x10, NT 10x4096x1024."""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
s = torch.cuda.current_stream().cuda_stream
A = torch.rand(4096 * 4096, device="cuda"); B = torch.rand(4096 * 4096, device="cuda"); C = torch.empty(4096 * 4096, device="cuda")
for rep in range(3):
    _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), 1024, 10, 4096, 0, s))
    _lib.check(L.mtnn_gemm_nn(A.data_ptr(), B.data_ptr(), C.data_ptr(), 1024, 4096, 10, 0, s))
    _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), 10, 4096, 1024, 0, s))
torch.cuda.synchronize()
print("ok")
