"""Each FCN-step call once (after one warm pass), for ncu launch lists:
ncu --metrics gpu__time_duration.sum,... python tools/probes/fcn_calls_once.py"""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
s = torch.cuda.current_stream().cuda_stream
widths = [784, 4096, 4096, 4096, 10]
layers = list(zip(widths[:-1], widths[1:]))
calls = [("nt", 1024, dout, din) for din, dout in layers]
for din, dout in reversed(layers):
    calls.append(("nn", 1024, din, dout)); calls.append(("nt", dout, din, 1024))
A = torch.rand(4096 * 4096, device="cuda") * 2 - 1; B = torch.rand(4096 * 4096, device="cuda") * 2 - 1
C = torch.empty(4096 * 4096, device="cuda")
for rep in range(2):
    for (op, m, n, k) in calls:
        fn = L.mtnn_gemm_nt if op == "nt" else L.mtnn_gemm_nn
        _lib.check(fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s))
    torch.cuda.synchronize()
print("ok")
