import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
torch.manual_seed(0)
for k in (256, 512, 1024, 2048, 4096, 8192):
    m = n = 2048 + 1024  # 24 x 12 = 288 tiles -> no split-K
    a = torch.rand(m, k, device=dev) * 2 - 1; b = torch.rand(n, k, device=dev) * 2 - 1
    want = a.double() @ b.double().t()
    c = torch.empty(m, n, device=dev)
    _lib.check(L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, 1, s)); torch.cuda.synchronize()
    d = c.double() - want
    rel = float(d.norm() / want.norm())
    bias = float((d * want.sign()).mean() / want.abs().mean())
    # positive-only data: all products positive, partial sums grow monotonically
    ap = torch.rand(m, k, device=dev); bp = torch.rand(n, k, device=dev)
    wp = ap.double() @ bp.double().t()
    _lib.check(L.mtnn_gemm_nt(ap.data_ptr(), bp.data_ptr(), c.data_ptr(), m, n, k, 1, s)); torch.cuda.synchronize()
    dp = c.double() - wp
    print(f"k={k}: rel={rel:.3e} signed-bias={bias:.3e} | positive data rel={float(dp.norm()/wp.norm()):.3e} mean rel={float((dp/wp).mean()):.3e}")
print("NN path:")
for k in (256, 4096, 16384):
    m = n = 2048
    a = torch.rand(m, k, device=dev) * 2 - 1; b = torch.rand(n, k, device=dev) * 2 - 1
    want = a.double() @ b.double().t(); bt = b.t().contiguous()
    c = torch.empty(m, n, device=dev)
    _lib.check(L.mtnn_gemm_nn(a.data_ptr(), bt.data_ptr(), c.data_ptr(), m, n, k, 1, s)); torch.cuda.synchronize()
    print(f"NN k={k}: rel={float((c.double()-want).norm()/want.norm()):.3e}")
    _lib.check(L.mtnn_gemm_tnn(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, 1, -1, s)); torch.cuda.synchronize()
    print(f"TNN k={k}: rel={float((c.double()-want).norm()/want.norm()):.3e}")
