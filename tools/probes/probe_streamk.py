"""Interleaved A/B of stream-K (knob tc_streamk) per shape (whole NT / NN calls:
split + GEMM + fix-up), then the whole configs[1] sweep total under each setting
(interleaved per case), then the FCN step. Modes: base = tc_streamk 0 (split-K
chooser, pairs as default); sk = tc_streamk 1 (auto); sk1 = tc_streamk 2 with
pairs off (stream-K single-CTA wherever possible)."""
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
flush = torch.ones(64 * 2**20, device=dev)
A = torch.rand(16384 * 16384, device=dev) * 2 - 1; B = torch.rand(16384 * 16384, device=dev) * 2 - 1
C = torch.empty(16384 * 16384, device=dev)
import os
MODES = {"base": (0, 1), "sk": (1, 1), "sk1": (2, 0)}
if os.environ.get("MODES"):
    MODES = {k: MODES[k] for k in os.environ["MODES"].split(",")}


def t_case(m, n, k, mode, op="nt", reps=5):
    sk, pair = MODES[mode]
    _lib.config_set("tc_streamk", sk); _lib.config_set("tc_pair", pair)
    fn = L.mtnn_gemm_nt if op == "nt" else L.mtnn_gemm_nn
    ev = []
    for rep in range(reps + 1):
        flush.sum(); torch.cuda._sleep(200000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _lib.check(fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, s)); b.record()
        if rep: ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


shapes = [("nt", 1024, 4096, 784), ("nt", 1024, 4096, 4096), ("nt", 4096, 4096, 1024), ("nt", 4096, 784, 1024),
          ("nn", 1024, 4096, 4096), ("nn", 1024, 784, 4096), ("nt", 4096, 4096, 4096), ("nt", 2048, 4096, 8192),
          ("nt", 8192, 4096, 2048), ("nt", 1024, 1024, 16384), ("nt", 2048, 2048, 4096), ("nt", 4096, 8192, 1024),
          ("nt", 512, 4096, 4096), ("nt", 8192, 8192, 1024), ("nt", 2048, 2048, 2048)]
for op, m, n, k in shapes:
    r = {}
    for rep in range(3):
        for mode in MODES:
            r.setdefault(mode, []).append(t_case(m, n, k, mode, op, reps=3))
    t = {md: min(v) for md, v in r.items()}
    f = 2 * m * n * k / 1e9
    print(f"{op} ({m},{n},{k}) " + " | ".join(f"{md} {t[md]*1e3:.1f} us {f/t[md]:.0f} TF/s" for md in MODES)
          + (f" | sk/base {t['base']/t['sk']:.3f}x" if "sk" in t and "base" in t else ""), flush=True)
if len(sys.argv) > 1 and sys.argv[1] == "sweep":
    E = [2 ** e for e in range(7, 15)]
    tot = {"base": 0.0, "sk": 0.0}
    for m in E:
        for n in E:
            for k in E:
                for mode in tot:
                    tot[mode] += t_case(m, n, k, mode, reps=2)
    F = 2 * 32640 ** 3
    print("sweep " + "  ".join(f"{md} {v:.1f} ms ({F/v/1e9:.0f} TF/s)" for md, v in tot.items()), flush=True)
