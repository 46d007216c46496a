"""Per-case breakdown of the MTNN sweep (configs[1]): total event time vs the
library's per-kernel-class times (split / gemm / reduce / transpose) and the
remainder (launch gaps). Writes gpurun_out/sweep_breakdown.csv."""
import csv, statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
E = [2 ** e for e in range(7, 15)]
shapes = [(m, n, k) for m in E for n in E for k in E]
variant = int(sys.argv[1]) if len(sys.argv) > 1 else 0
if len(sys.argv) > 2:
    _lib.config_set("f16s_inkernel_max_short", int(sys.argv[2]))
tag = "_".join(sys.argv[1:]) or "0"
A = torch.rand(16384 * 16384, device=dev) * 2 - 1
B = torch.rand(16384 * 16384, device=dev) * 2 - 1
C = torch.empty(16384 * 16384, device=dev)
rows = []
tot = {}
for (m, n, k) in shapes:
    f = lambda: _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, variant, s))
    f()
    L.mtnn_profile_reset(); L.mtnn_profile_enable(1)
    ev = []
    for _ in range(3):
        flush.sum(); torch.cuda._sleep(200000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    L.mtnn_profile_enable(0)
    t = statistics.median(a.elapsed_time(b) for a, b in ev)
    prof = {_lib.KCLASS_NAMES[c]: _lib.profile_read(c)[0] / 3 for c in _lib.KCLASS_NAMES}
    gemm = prof["gemm_tc3xf16s"] + prof["gemm_tc3xtf32"] + prof["gemm_ffma"]
    row = dict(m=m, n=n, k=k, total_ms=t, gemm_ms=gemm, split_ms=prof["operand_split"],
               reduce_ms=prof["splitk_reduce"], gap_ms=t - gemm - prof["operand_split"] - prof["splitk_reduce"])
    rows.append(row)
with open(f"gpurun_out/sweep_breakdown_{tag}.csv", "w", newline="") as fh:
    w = csv.DictWriter(fh, fieldnames=list(rows[0])); w.writeheader(); w.writerows(rows)
T = sum(r["total_ms"] for r in rows)
F = sum(2.0 * r["m"] * r["n"] * r["k"] for r in rows)
print(f"args {sys.argv[1:]}: total {T:.2f} ms -> {F / T / 1e9:.1f} TF/s")
for key in ("gemm_ms", "split_ms", "reduce_ms", "gap_ms"):
    print(f"  {key}: {sum(r[key] for r in rows):.2f} ms")
