"""Per-call device time of the FCN step (configs[3]) by variant."""
import statistics, sys, torch
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
tot = {}
for (op, m, n, k) in calls:
    out = []
    for v in (0, 2, 1, 3):
        fn = L.mtnn_gemm_nt if op == "nt" else L.mtnn_gemm_nn
        ev = []
        ok = True
        for rep in range(6):
            flush.sum(); torch.cuda._sleep(100000)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); rc = fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, v, s); b.record()
            if rc: ok = False; break
            if rep: ev.append((a, b))
        torch.cuda.synchronize()
        t = statistics.median(a.elapsed_time(b) for a, b in ev) * 1e3 if ok else float("nan")
        tot[v] = tot.get(v, 0) + (t if ok else 0)
        out.append(f"v{v} {t:7.1f}us")
    print(f"{op} ({m},{n},{k}) " + "  ".join(out), flush=True)
print("totals", tot)
