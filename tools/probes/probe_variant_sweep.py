"""Per-shape timings of the tc3xf16s variant decisions over the configs[1]
sweep (m, n, k in 2^7..2^14), interleaved per case, median of 5, L2 flushed:
  pair: single-CTA 128x256 tiles (tc_pair 0) vs CTA pairs 256x256 (tc_pair 2),
        shapes with m, n > 128;
  ink:  pre-split operands (f16s_inkernel_max_short 0) vs the long operand
        split inside the GEMM (max_short 512), shapes with short side <= 512
        and long side >= 1024.
Writes gpurun_out/variants.csv (m, n, k, decision, t0, t1)."""
import csv, statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
A = torch.rand(16384 * 16384, device=dev) * 2 - 1; B = torch.rand(16384 * 16384, device=dev) * 2 - 1
C = torch.empty(16384 * 16384, device=dev)
old_pair, old_ink = _lib.config_get("tc_pair"), _lib.config_get("f16s_inkernel_max_short")


def run(m, n, k):
    _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 3, s))


def timed(m, n, k, setting):
    for key, v in setting.items():
        _lib.config_set(key, v)
    flush.sum(); torch.cuda._sleep(100000)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); run(m, n, k); b.record()
    return a, b


E = [2 ** e for e in range(7, 15)]
rows = []
for m in E:
    for n in E:
        for k in E:
            decisions = []
            if m > 128 and n > 128:
                decisions.append(("pair", {"tc_pair": 0, "f16s_inkernel_max_short": old_ink},
                                  {"tc_pair": 2, "f16s_inkernel_max_short": old_ink}))
            if min(m, n) <= 512 and max(m, n) >= 1024:
                decisions.append(("ink", {"tc_pair": old_pair, "f16s_inkernel_max_short": 0},
                                  {"tc_pair": old_pair, "f16s_inkernel_max_short": 512}))
            for name, s0, s1 in decisions:
                ev = {0: [], 1: []}
                run(m, n, k)
                for rep in range(5):
                    for v, st in ((0, s0), (1, s1)) if rep % 2 == 0 else ((1, s1), (0, s0)):
                        ev[v].append(timed(m, n, k, st))
                torch.cuda.synchronize()
                t0 = statistics.median(a.elapsed_time(b) for a, b in ev[0]) * 1e-3
                t1 = statistics.median(a.elapsed_time(b) for a, b in ev[1]) * 1e-3
                rows.append(dict(m=m, n=n, k=k, decision=name, t0=t0, t1=t1))
_lib.config_set("tc_pair", old_pair); _lib.config_set("f16s_inkernel_max_short", old_ink)
with open("gpurun_out/variants.csv", "w", newline="") as fh:
    w = csv.DictWriter(fh, fieldnames=list(rows[0])); w.writeheader(); w.writerows(rows)
for name in ("pair", "ink"):
    r = [x for x in rows if x["decision"] == name]
    print(name, len(r), "cases; variant 1 wins", sum(x["t1"] < x["t0"] for x in r),
          "; sum t0 %.1f ms, t1 %.1f ms, best %.1f ms" % (sum(x["t0"] for x in r) * 1e3,
          sum(x["t1"] for x in r) * 1e3, sum(min(x["t0"], x["t1"]) for x in r) * 1e3))
