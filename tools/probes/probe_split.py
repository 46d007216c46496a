"""Split-kernel time per operand shape (one launch for A and B), interleaved."""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
A = torch.rand(16384 * 16384, device=dev); B = torch.rand(16384 * 16384, device=dev); C = torch.empty(16384 * 16384, device=dev)
tot = 0.0
import os
shapes = [(2048, 2048, 2048), (4096, 4096, 1024), (8192, 8192, 512), (16384, 16384, 2048), (1024, 1024, 1024), (512, 8192, 256)]
if os.environ.get('SHORTK'):
    shapes = [(2048, 2048, 2048), (4096, 4096, 1024), (8192, 8192, 512), (16384, 16384, 2048), (1024, 1024, 1024), (512, 8192, 256), (16384, 16384, 1024), (16384, 16384, 512), (16384, 16384, 256), (4096, 4096, 256)]
if os.environ.get('LONGK'):
    shapes = [(8192, 8192, 8192), (16384, 16384, 16384), (4096, 4096, 4096), (16384, 8192, 8192), (128, 16384, 16384), (2048, 2048, 8192)]
for (m, n, k) in shapes:
    _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 3, s))  # warm (lazy module load)
    torch.cuda.synchronize()
    L.mtnn_profile_reset(); L.mtnn_profile_enable(1)
    for rep in range(5):
        flush.sum(); torch.cuda._sleep(100000)
        _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 3, s))
    torch.cuda.synchronize(); L.mtnn_profile_enable(0)
    ms, nl, w = _lib.profile_read(_lib.KCLASS_SPLIT)
    print(f"({m},{n},{k}) split {ms/5*1e3:.1f} us  {w/(ms*1e-3)/1e9:.0f} GB/s", flush=True)
