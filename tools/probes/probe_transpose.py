import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
B = torch.rand(16384 * 16384, device=dev); C = torch.empty(16384 * 16384, device=dev)
for (r, c) in [(4097, 1023), (12345, 6789), (8191, 8193), (1000, 1000), (3000, 5000), (16384, 16384), (8192, 8192), (4096, 4096), (1001, 16385), (16384, 128), (128, 16384), (16384, 256), (65536, 64), (64, 65536), (262144, 64), (64, 262144), (131072, 128), (524288, 32)]:
    ev = []
    for rep in range(6):
        flush.sum(); torch.cuda._sleep(100000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _lib.check(L.mtnn_transpose(B.data_ptr(), C.data_ptr(), r, c, s)); b.record()
        if rep: ev.append((a, b))
    torch.cuda.synchronize()
    t = statistics.median(x.elapsed_time(y) for x, y in ev) * 1e-3
    ok = torch.equal(C[: r * c].view(c, r), B[: r * c].view(r, c).t())
    print(f"{r}x{c}: {8*r*c/t/1e9:.0f} GB/s exact={ok}", flush=True)
