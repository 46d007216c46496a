"""Phase timeline of the single-CTA tensor-core GEMM (mtnn_profile_trace): per
phase, the median / max over CTAs of globaltimer ns since the first CTA's entry.
Whole calls (split -> GEMM -> fix-up, chained), warm, one after another."""
import os, statistics, sys, torch
sys.path.insert(0, ".")
# phase traces need a -DMTNN_TRACE build: tools/build_variant.sh trace -DMTNN_TRACE
os.environ.setdefault("MTNN_B200_LIB", "build/variants/trace/libmtnn_b200.so")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
_lib.config_set("tc_pair", 0)
import os
NAMES = ["entry", "prologue", "pdl_wait", "tma0", "stage0", "mma_last", "chunk0", "chunk_last",
         "stores_issued", "stores_done", "exit", "tma_last", "producer_w0", "last_promoted", "first_store_issued"]
A = torch.rand(4096 * 16384, device=dev); B = torch.rand(4096 * 16384, device=dev); C = torch.empty(4096 * 4096, device=dev)
tr = torch.zeros(148 * 16, dtype=torch.int64, device=dev)
shapes = [(1024, 4096, k) for k in (512, 4096)] + [(2048, 2048, 1024), (4096, 4096, 4096), (256, 4096, 4096)]
if os.environ.get("SHAPES"):
    shapes = [tuple(int(x) for x in t.split("x")) for t in os.environ["SHAPES"].split(",")]
for m, n, k in shapes:
    for _ in range(3):
        _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 3, s))
    torch.cuda.synchronize()
    tr.zero_()
    _lib.check(L.mtnn_profile_trace(tr.data_ptr(), 148))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 3, s))
    ev[1].record()
    torch.cuda.synchronize()
    _lib.check(L.mtnn_profile_trace(None, 0))
    t = tr.view(148, 16).cpu().numpy()
    rows = [r for r in t if r[0] != 0]
    t0 = min(r[0] for r in rows)
    mma = 2 * m * n * k / 1e3  # flop per ns at 1 PF/s... just for context
    print(f"({m},{n},{k}) CTAs {len(rows)}, call window {ev[0].elapsed_time(ev[1])*1e3:.1f} us")
    for i, nm in enumerate(NAMES):
        v = [(r[i] - t0) / 1e3 for r in rows if r[i] != 0]
        if v:
            print(f"   {nm:14s} med {statistics.median(v):8.2f} us  min {min(v):8.2f}  max {max(v):8.2f}")
