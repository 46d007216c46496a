"""PCIe duplex: H2D (contiguous) concurrent with D2H (contiguous or 2-D with
narrower rows), rates of each direction from CUDA events on their streams."""
import torch
import cuda.bindings.runtime as rt
dev = torch.device("cuda:0")
N = 64 * 2**20  # floats per buffer (256 MB)
h_in = torch.empty(N, dtype=torch.float32).pin_memory()
h_out = torch.empty(N, dtype=torch.float32).pin_memory()
d_in = torch.empty(N, device=dev); d_out = torch.empty(N, device=dev)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
def d2h(width_f, pitch_f):
    rows = N // pitch_f
    err, = rt.cudaMemcpy2DAsync(h_out.data_ptr(), pitch_f * 4, d_out.data_ptr(), width_f * 4, width_f * 4,
                                rows, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s_out.cuda_stream)
    return rows * width_f * 4
def run(h2d, width_f, pitch_f):
    torch.cuda.synchronize()
    ei = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    eo = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    bi = bo = 0
    if h2d:
        ei[0].record(s_in)
        with torch.cuda.stream(s_in):
            d_in.copy_(h_in, non_blocking=True)
        ei[1].record(s_in); bi = 4 * N
    if width_f:
        eo[0].record(s_out); bo = d2h(width_f, pitch_f); eo[1].record(s_out)
    torch.cuda.synchronize()
    ri = bi / ei[0].elapsed_time(ei[1]) / 1e6 if h2d else 0
    ro = bo / eo[0].elapsed_time(eo[1]) / 1e6 if width_f else 0
    return ri, ro
for _ in range(2):
    print("H2D alone           %.1f GB/s" % run(True, 0, 0)[0])
    print("D2H alone contig    %.1f GB/s" % run(False, 16384, 16384)[1])
    for w in (16384, 4096, 1536, 1024, 512):
        print("D2H alone 2-D w=%6d B  %.1f GB/s" % (4 * w, run(False, w, 16384)[1]))
    for w in (16384, 4096, 1536, 1024):
        ri, ro = run(True, w, 16384)
        print("duplex: H2D %.1f GB/s  D2H 2-D w=%6d B %.1f GB/s  sum %.1f" % (ri, 4 * w, ro, ri + ro))
# closer to the blocked pipeline: 25 MB pieces each way, optionally with a
# tensor-core GEMM (torch fp32 8192^3) and an HBM-bound kernel on a third stream
def pieces(compute):
    s_c = torch.cuda.Stream()
    x = torch.rand(8192, 8192, device=dev)
    torch.cuda.synchronize()
    ei = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    eo = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    P = 6 * 2**20  # floats per piece (25 MB)
    ei[0].record(s_in); eo[0].record(s_out)
    if compute:
        with torch.cuda.stream(s_c):
            for _ in range(6):
                y = x @ x
    for i in range(10):
        with torch.cuda.stream(s_in):
            d_in[i * P:(i + 1) * P].copy_(h_in[i * P:(i + 1) * P], non_blocking=True)
        rt.cudaMemcpy2DAsync(h_out.data_ptr() + 4 * 1536 * i, 16384 * 4, d_out.data_ptr() + 4 * P * i, 1536 * 4,
                             1536 * 4, 4096, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s_out.cuda_stream)
    ei[1].record(s_in); eo[1].record(s_out)
    torch.cuda.synchronize()
    return 10 * 4 * P / ei[0].elapsed_time(ei[1]) / 1e6, 10 * 4 * 1536 * 4096 / eo[0].elapsed_time(eo[1]) / 1e6
for c in (False, True, False, True):
    ri, ro = pieces(c)
    print("pieces%s: H2D %.1f GB/s  D2H 2-D 6 KB rows %.1f GB/s" % (" + GEMM" if c else "", ri, ro))
