import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
torch.manual_seed(0)
def rel(c, w): return float((c.double() - w).norm() / w.norm())
print("== correctness / accuracy (variant 3 = tc3xf16s, 1 = tc3xtf32)")
for (m, n, k, kind) in [(128, 256, 32, "u"), (256, 512, 128, "u"), (200, 304, 104, "u"), (1000, 1008, 1000, "u"),
                        (3000, 2048, 4096, "u"), (2048, 2048, 4096, "pos"), (2048, 2048, 4096, "wide"),
                        (2048, 2048, 16384, "u"), (128, 128, 16384, "u"), (16384, 128, 1024, "u")]:
    if kind == "u":
        a = torch.rand(m, k, device=dev) * 2 - 1; b = torch.rand(n, k, device=dev) * 2 - 1
    elif kind == "pos":
        a = torch.rand(m, k, device=dev); b = torch.rand(n, k, device=dev)
    else:
        a = torch.randn(m, k, device=dev) * torch.exp(torch.empty(m, 1, device=dev).uniform_(-40, 40))
        b = torch.randn(n, k, device=dev) * torch.exp(torch.empty(n, 1, device=dev).uniform_(-20, 20))
    want = a.double() @ b.double().t()
    bt = b.t().contiguous()
    out = []
    for v in (3, 1):
        c = torch.full((m, n), float("nan"), device=dev)
        _lib.check(L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, v, s))
        c2 = torch.full((m, n), float("nan"), device=dev)
        _lib.check(L.mtnn_gemm_nn(a.data_ptr(), bt.data_ptr(), c2.data_ptr(), m, n, k, v, s))
        torch.cuda.synchronize()
        out.append(f"v{v}: nt {rel(c, want):.2e} nn {rel(c2, want):.2e}")
    print(f"({m},{n},{k}) {kind}: " + " | ".join(out))

def bench(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(iters): fn()
    en.record(); torch.cuda.synchronize()
    return st.elapsed_time(en) / iters * 1e-3
print("== perf (TFLOP/s incl. split)")
for (m, n, k) in [(1024, 1024, 1024), (4096, 4096, 4096), (8192, 8192, 8192), (16384, 16384, 16384), (16384, 16384, 1024), (16384, 128, 16384), (128, 16384, 16384)]:
    a = torch.rand(m, k, device=dev); b = torch.rand(n, k, device=dev); c = torch.empty(m, n, device=dev)
    bt = b.t().contiguous()
    row = []
    for v in (3, 1):
        t = bench(lambda: L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, v, s))
        t2 = bench(lambda: L.mtnn_gemm_nn(a.data_ptr(), bt.data_ptr(), c.data_ptr(), m, n, k, v, s))
        t3 = bench(lambda: L.mtnn_gemm_tnn(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, v, -1, s))
        f = 2 * m * n * k / 1e12
        row.append(f"v{v}: NT {f/t:.0f} NN {f/t2:.0f} TNN {f/t3:.0f}")
    print(f"({m},{n},{k}) " + " | ".join(row))
# kernel-only time via profile counters
L.mtnn_profile_reset(); L.mtnn_profile_enable(1)
m = n = k = 8192
a = torch.rand(m, k, device=dev); b = torch.rand(n, k, device=dev); c = torch.empty(m, n, device=dev)
for v in (3,):
    for _ in range(5): L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, v, s)
torch.cuda.synchronize(); L.mtnn_profile_enable(0)
for cl in range(5):
    ms, nl, w = _lib.profile_read(cl)
    if nl: print(_lib.KCLASS_NAMES[cl], f"{ms/nl:.3f} ms/launch", f"{w/ (ms*1e-3)/1e12:.1f} T/s" if cl < 2 else f"{w/(ms*1e-3)/1e9:.0f} GB/s")
