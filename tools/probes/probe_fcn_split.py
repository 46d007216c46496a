"""Per-call split / GEMM kernel times of the FCN step (configs[3]) on the
tc3xf16s path: which operand split is far from the HBM roof."""
import sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
widths = [784, 4096, 4096, 4096, 10]
layers = list(zip(widths[:-1], widths[1:]))
calls = [("nt", 1024, dout, din) for din, dout in layers]
for din, dout in reversed(layers):
    calls.append(("nn", 1024, din, dout)); calls.append(("nt", dout, din, 1024))
A = torch.rand(4096 * 4096, device=dev); B = torch.rand(4096 * 4096, device=dev); C = torch.empty(4096 * 4096, device=dev)
tot_s = tot_g = 0.0
for (op, m, n, k) in calls:
    fn = L.mtnn_gemm_nt if op == "nt" else L.mtnn_gemm_nn
    fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)
    torch.cuda.synchronize()
    L.mtnn_profile_reset(); L.mtnn_profile_enable(1)
    for rep in range(5):
        flush.sum(); torch.cuda._sleep(100000)
        fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)
    torch.cuda.synchronize(); L.mtnn_profile_enable(0)
    ms, nl, w = _lib.profile_read(_lib.KCLASS_SPLIT)
    gms, gnl, gw = _lib.profile_read(_lib.KCLASS_GEMM_TC_F16S)
    tot_s += ms / 5; tot_g += gms / 5
    print(f"{op} ({m},{n},{k}) split {ms/5*1e3:6.1f} us x{nl//5} {w/max(ms,1e-9)/1e6:5.0f} GB/s | "
          f"gemm {gms/5*1e3:6.1f} us {gw/max(gms,1e-9)/1e9:5.0f} TF/s", flush=True)
print(f"total split {tot_s*1e3:.1f} us, gemm {tot_g*1e3:.1f} us")
