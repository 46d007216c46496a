"""Per-case end-to-end (host buffers) time of the sweep vs the PCIe floor."""
import csv, ctypes, sys, time, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
E = [2 ** e for e in range(7, 15)]
shapes = [(m, n, k) for m in E for n in E for k in E]
ha = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hb = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory().uniform_(-1, 1)
hc = torch.empty(16384 * 16384, dtype=torch.float32).pin_memory()
rows = []
for (m, n, k) in shapes:
    ts = []
    for rep in range(3):
        t0 = time.perf_counter()
        _lib.check(L.mtnn_gemm_nt_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, 0))
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[1]
    h2d, d2h = 4 * (m * k + n * k), 4 * m * n
    floor = max(h2d / 55.5e9, d2h / 54.2e9)
    rows.append(dict(m=m, n=n, k=k, t=t, floor=floor, h2d=h2d, d2h=d2h))
import os
with open(os.environ.get("OUT", "gpurun_out/e2e_cases.csv"), "w", newline="") as fh:
    w = csv.DictWriter(fh, fieldnames=list(rows[0])); w.writeheader(); w.writerows(rows)
T = sum(r["t"] for r in rows); Fl = sum(r["floor"] for r in rows)
print(f"total {T*1e3:.1f} ms floor {Fl*1e3:.1f} ms  TF/s {2*32640**3/T/1e12:.1f}")
