"""Quick GPU probe: correctness + timing of every kernel through the device C-ABI."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib

def cptr(t): return t.data_ptr()

def relfro(got, want):
    got = got.double(); want = want.double()
    return float((got - want).norm() / want.norm().clamp_min(1e-300))

torch.manual_seed(0)
dev = torch.device("cuda:0")
s = torch.cuda.current_stream().cuda_stream
print("features", end=" ")
import ctypes
f = (ctypes.c_double * 5)(); _lib.check(L.mtnn_device_features(f)); print(list(f))

# transpose
for (r, c) in [(1, 1), (2, 3), (37, 65), (128, 128), (1000, 1000), (4097, 1023), (3000, 5000), (8191, 8193), (4096, 4096)]:
    b = torch.randint(-2**31, 2**31 - 1, (r, c), dtype=torch.int32, device=dev).view(torch.float32)
    bt = torch.empty((c, r), dtype=torch.float32, device=dev)
    _lib.check(L.mtnn_transpose(cptr(b), cptr(bt), r, c, s))
    torch.cuda.synchronize()
    ok = torch.equal(bt.view(torch.int32), b.view(torch.int32).t().contiguous())
    print(f"transpose {r}x{c}: bitexact={ok}")

for variant in (2, 1):
    for (m, n, k) in [(1, 1, 1), (3, 5, 7), (64, 64, 64), (128, 256, 16), (128, 256, 32), (128, 256, 64), (256, 512, 128), (200, 300, 100), (1024, 1024, 1024), (130, 260, 36), (128, 128, 16384), (4096, 4096, 4096)]:
        if variant == 1 and (k % 4 or n % 4): continue
        a = torch.rand(m, k, device=dev) * 2 - 1
        b = torch.rand(n, k, device=dev) * 2 - 1
        want = a.double() @ b.double().t()
        c = torch.full((m, n), float("nan"), device=dev)
        rc = L.mtnn_gemm_nt(cptr(a), cptr(b), cptr(c), m, n, k, variant, s)
        if rc: print("nt err", _lib.last_error()); continue
        torch.cuda.synchronize()
        e_nt = relfro(c, want)
        bt = b.t().contiguous()
        c2 = torch.full((m, n), float("nan"), device=dev)
        e_nn = None
        if variant == 2 or n % 16 == 0:
            rc = L.mtnn_gemm_nn(cptr(a), cptr(bt), cptr(c2), m, n, k, variant, s)
            if rc: print("nn err", _lib.last_error())
            torch.cuda.synchronize()
            e_nn = relfro(c2, want)
        print(f"variant={variant} ({m},{n},{k}) nt_err={e_nt:.3e} nn_err={e_nn}")

# timings
def bench(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(iters): fn()
    en.record(); torch.cuda.synchronize()
    return st.elapsed_time(en) / iters * 1e-3

for (m, n, k) in [(1024, 1024, 1024), (4096, 4096, 4096), (8192, 8192, 8192), (128, 128, 16384), (16384, 16384, 128)]:
    a = torch.rand(m, k, device=dev); b = torch.rand(n, k, device=dev); c = torch.empty(m, n, device=dev)
    bt = b.t().contiguous()
    for variant in (1, 2):
        t = bench(lambda: L.mtnn_gemm_nt(cptr(a), cptr(b), cptr(c), m, n, k, variant, s))
        t2 = bench(lambda: L.mtnn_gemm_nn(cptr(a), cptr(bt), cptr(c), m, n, k, variant, s))
        t3 = bench(lambda: L.mtnn_gemm_tnn(cptr(a), cptr(b), cptr(c), m, n, k, variant, -1, s))
        print(f"({m},{n},{k}) v{variant}: NT {2*m*n*k/t/1e12:.1f} TF  NN {2*m*n*k/t2/1e12:.1f} TF  TNN {2*m*n*k/t3/1e12:.1f} TF")
torch.backends.cuda.matmul.allow_tf32 = False
a = torch.rand(8192, 8192, device=dev); b = torch.rand(8192, 8192, device=dev)
t = bench(lambda: a @ b.t()); print(f"torch fp32 (cuBLAS) 8192^3 NT: {2*8192**3/t/1e12:.1f} TF")
torch.backends.cuda.matmul.allow_tf32 = True
t = bench(lambda: a @ b.t()); print(f"torch tf32 (cuBLAS) 8192^3 NT: {2*8192**3/t/1e12:.1f} TF")
for r in (4096, 16384):
    b = torch.rand(r, r, device=dev); bt = torch.empty_like(b)
    t = bench(lambda: L.mtnn_transpose(cptr(b), cptr(bt), r, r, s))
    print(f"transpose {r}^2: {8*r*r/t/1e9:.0f} GB/s")
    t = bench(lambda: bt.copy_(b))
    print(f"copy {r}^2: {8*r*r/t/1e9:.0f} GB/s")
