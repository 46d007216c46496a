import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
torch.manual_seed(0)
def rel(c, w): return float((c.double() - w).norm() / w.norm())
flush = torch.ones(64 * 2**20, device=dev)
def bench(fn, iters=5):
    ts = []
    for _ in range(2): fn()
    for _ in range(iters):
        flush.sum(); torch.cuda._sleep(200000)
        st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
        st.record(); fn(); en.record()
        ts.append((st, en))
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ts)[iters // 2] * 1e-3
print("shape | err v1 v3 | TF: auto, tf32(in-kernel), f16s")
for (m, n, k) in [(16384, 128, 16384), (128, 16384, 16384), (8192, 128, 4096), (16384, 512, 16384), (4096, 256, 16384), (16384, 16384, 128), (2048, 2048, 2048), (8192, 8192, 8192), (300, 2048, 1000)]:
    a = torch.rand(m, k, device=dev) * 2 - 1; b = torch.rand(n, k, device=dev) * 2 - 1
    c = torch.empty(m, n, device=dev); bt = b.t().contiguous()
    errs = []
    if m * n <= 2**27:
        want = a.double() @ b.double().t()
        for v in (1, 3):
            _lib.check(L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, v, s)); torch.cuda.synchronize()
            errs.append(f"{rel(c, want):.1e}")
            if n % 16 == 0:
                _lib.check(L.mtnn_gemm_nn(a.data_ptr(), bt.data_ptr(), c.data_ptr(), m, n, k, v, s)); torch.cuda.synchronize()
                errs.append(f"nn{rel(c, want):.1e}")
    tf = []
    for v in (0, 1, 3):
        t = bench(lambda: L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, v, s))
        tf.append(f"{2*m*n*k/t/1e12:.0f}")
    print(f"({m},{n},{k}) | {' '.join(errs)} | {' '.join(tf)}", flush=True)
