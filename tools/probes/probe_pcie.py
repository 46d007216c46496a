import time, torch
dev = torch.device("cuda:0")
N = 256 * 2**20  # 1 GiB of fp32
h = torch.empty(N, dtype=torch.float32).pin_memory(); h.uniform_()
h2 = torch.empty(N, dtype=torch.float32).pin_memory()
d = torch.empty(N, device=dev); d2 = torch.empty(N, device=dev)
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
gb = N * 4 / 1e9
print("H2D GB/s", gb / t(lambda: d.copy_(h, non_blocking=True)))
print("D2H GB/s", gb / t(lambda: h2.copy_(d, non_blocking=True)))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print("H2D+D2H concurrent GB/s each", gb / t(both))
def two_h2d():
    with torch.cuda.stream(s1): d[: N // 2].copy_(h[: N // 2], non_blocking=True)
    with torch.cuda.stream(s2): d[N // 2:].copy_(h[N // 2:], non_blocking=True)
print("H2D two streams GB/s", gb / t(two_h2d))
for mb in (1, 4, 16, 64):
    n = mb * 2**18
    print(f"H2D {mb} MiB chunk GB/s", n * 4 / 1e9 / t(lambda: d[:n].copy_(h[:n], non_blocking=True), reps=20))
import os; print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
