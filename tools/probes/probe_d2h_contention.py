"""D2H (2-D, 6 KB rows, 100 MB) alone and concurrent with: an HBM copy kernel,
our tensor-core GEMM (device API), a torch fp32 GEMM."""
import ctypes, sys, torch
import cuda.bindings.runtime as rt
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0")
N = 64 * 2**20
h_out = torch.empty(N, dtype=torch.float32).pin_memory()
d_out = torch.empty(N, device=dev)
s_out, s_c = torch.cuda.Stream(), torch.cuda.Stream()
big = torch.rand(256 * 2**20 // 4 * 4, device=dev); big2 = torch.empty_like(big)
a = torch.rand(8192, 8192, device=dev); b = torch.rand(8192, 8192, device=dev); c = torch.empty(8192, 8192, device=dev)
def d2h_rate(load):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_c):
        for _ in range(12):
            if load == "copy": big2.copy_(big)
            elif load == "mtnn": _lib.check(L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), 8192, 8192, 8192, 0, s_c.cuda_stream))
            elif load == "torch": torch.mm(a, b, out=c)
    e0.record(s_out)
    for i in range(4):
        rt.cudaMemcpy2DAsync(h_out.data_ptr() + 4 * 1536 * i, 16384 * 4, d_out.data_ptr(), 1536 * 4, 1536 * 4, 4096,
                             rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s_out.cuda_stream)
    e1.record(s_out)
    torch.cuda.synchronize()
    return 4 * 4 * 1536 * 4096 / e0.elapsed_time(e1) / 1e6
for _ in range(2):
    for load in ("none", "copy", "mtnn", "torch"):
        print(f"D2H with {load:5s}: {d2h_rate(load):.1f} GB/s", flush=True)
