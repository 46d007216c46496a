"""Does a second read of an operand hit L2? Time x.amax() (a pure read) cold
(after a 256 MiB flush) and warm (right after a first read), for 16-128 MB."""
import statistics, torch
flush = torch.ones(64 * 2**20, device="cuda")
for mb in (16, 32, 48, 64, 80, 96, 128):
    x = torch.rand(mb * 2**18, device="cuda")
    cold, warm = [], []
    for _ in range(7):
        flush.sum(); torch.cuda._sleep(100000)
        e = [torch.cuda.Event(True) for _ in range(3)]
        e[0].record(); x.amax(); e[1].record(); x.amax(); e[2].record()
        torch.cuda.synchronize()
        cold.append(e[0].elapsed_time(e[1])); warm.append(e[1].elapsed_time(e[2]))
    c, w = statistics.median(cold), statistics.median(warm)
    print(f"{mb:4d} MB: cold {c*1e3:7.1f} us ({mb/1024/c*1e3:.2f} TB/s)  warm {w*1e3:7.1f} us "
          f"({mb/1024/w*1e3:.2f} TB/s)", flush=True)
