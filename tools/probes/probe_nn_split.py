import statistics, sys, os, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
A = torch.rand(16384 * 16384, device=dev); B = torch.rand(16384 * 16384, device=dev); C = torch.empty(16384 * 16384, device=dev)
tot = 0
for (m, n, k) in [(1024, 4096, 4096), (1024, 784, 4096), (4096, 4096, 4096), (8192, 8192, 2048), (2048, 16384, 1024), (4096, 8192, 8192), (1024, 4096, 784), (4096, 16384, 16384), (2048, 2048, 2048), (4096, 128, 4096)]:
    _lib.check(L.mtnn_gemm_nn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); torch.cuda.synchronize()
    ev = []; L.mtnn_profile_reset(); L.mtnn_profile_enable(1)
    for rep in range(6):
        flush.sum(); torch.cuda._sleep(100000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _lib.check(L.mtnn_gemm_nn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); b.record()
        if rep: ev.append((a, b))
    torch.cuda.synchronize(); L.mtnn_profile_enable(0)
    t = statistics.median(x.elapsed_time(y) for x, y in ev) * 1e3
    sp = _lib.profile_read(_lib.KCLASS_SPLIT)[0] / 6 * 1e3
    print(f"strip={os.environ.get('MTNN_SPLIT_STRIP','2')} nn ({m},{n},{k}) total {t:.1f} us split {sp:.1f} us", flush=True)
