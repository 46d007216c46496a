"""Does HBM traffic on the idle SMs slow a power-bound one-wave GEMM? A
1024x4096x4096 NT (128 CTAs on 148 SMs) alone vs with an HBM-bound transpose
stream on a second stream launched right after it; GEMM kernel time from
mtnn_profile_trace (entry of its first CTA -> last C store complete)."""
import os, statistics, sys, torch
sys.path.insert(0, ".")
# phase traces need a -DMTNN_TRACE build: tools/build_variant.sh trace -DMTNN_TRACE
os.environ.setdefault("MTNN_B200_LIB", "build/variants/trace/libmtnn_b200.so")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0")
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
_lib.config_set("tc_pair", 0)
A = torch.rand(4096 * 4096, device=dev); B = torch.rand(4096 * 4096, device=dev); C = torch.empty(4096 * 4096, device=dev)
X = torch.rand(16384 * 16384, device=dev); Y = torch.empty_like(X)
tr = torch.zeros(148 * 16, dtype=torch.int64, device=dev)
def run(concurrent):
    tr.zero_()
    torch.cuda.synchronize()
    with torch.cuda.stream(s2):
        torch.cuda._sleep(20000)
    with torch.cuda.stream(s1):
        _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), 1024, 4096, 4096, 3, s1.cuda_stream))
    if concurrent:
        with torch.cuda.stream(s2):
            for _ in range(2):
                _lib.check(L.mtnn_transpose(X.data_ptr(), Y.data_ptr(), 16384, 16384, s2.cuda_stream))
    torch.cuda.synchronize()
    t = tr.view(148, 16).cpu().numpy()
    rows = [r for r in t if r[0] != 0]
    t0 = min(r[2] for r in rows)  # after the dependency wait
    return (max(r[9] for r in rows) - t0) / 1e3
_lib.check(L.mtnn_profile_trace(tr.data_ptr(), 148))
for _ in range(3): run(False); run(True)
a = [run(False) for _ in range(7)]
b = [run(True) for _ in range(7)]
c = [run(False) for _ in range(7)]
print(f"GEMM alone {statistics.median(a):.1f} us, with concurrent transposes {statistics.median(b):.1f} us, alone again {statistics.median(c):.1f} us")
_lib.check(L.mtnn_profile_trace(None, 0))
