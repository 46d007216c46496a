"""Time the REAL reference (numba, from baseline/_ref) beside the oracle/ C
port that bench.py's CPU legs use, on the same shapes and thread counts, so the
port's speed relative to the reference is a committed measurement.

    python tools/ref_vs_port.py [out.json]

Cases: configs[0] (1024^3) and the 2^7..2^11 sweep sub-grid (125 cases), NT and
TNN, threads = 1 and all host cores; each timing is the median of 3 after one
warm call (numba JIT compiled before timing). Run it on the GPU box (the
bench's host) — baseline/_ref travels with gpurun.
"""
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_ref_vs_port")
os.environ["MTNN_BACKEND"] = "numba"

import oracle  # noqa: E402
from mtnn import bench as rbench  # noqa: E402  (the reference)
from mtnn import kernels as rk  # noqa: E402


def med(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def main(out_path="gpurun_out/ref_vs_port.json"):
    import numba

    cores = len(os.sched_getaffinity(0))
    nthreads = min(cores, numba.config.NUMBA_NUM_THREADS)
    res = {"host_cores": cores, "numba_threads": nthreads, "numba": numba.__version__, "cases": {}}
    sub = [(m, n, k) for m in (128, 256, 512, 1024, 2048) for n in (128, 256, 512, 1024, 2048)
           for k in (128, 256, 512, 1024, 2048)]
    for threads in (1, nthreads):
        tot = {"ref_nt": 0.0, "ref_tnn": 0.0, "port_nt": 0.0, "port_tnn": 0.0, "flops": 0.0}
        for (m, n, k) in [(1024, 1024, 1024)] + sub:
            a, b, _ = rbench.make_operands(rk.ProblemShape(m, n, k), 0)
            t = {
                "ref_nt": med(lambda: rk.gemm_nt(a, b, threads=threads)),
                "ref_tnn": med(lambda: rk.gemm_tnn(a, b, threads=threads)),
                "port_nt": med(lambda: oracle.gemm_nt(a, b, threads=threads)),
                "port_tnn": med(lambda: oracle.gemm_tnn(a, b, threads=threads)),
            }
            if (m, n, k) == (1024, 1024, 1024):
                res["cases"][f"1024^3 threads={threads}"] = {kk: v * 1e3 for kk, v in t.items()}
                res["cases"][f"1024^3 threads={threads}"]["unit"] = "ms"
                continue
            for kk, v in t.items():
                tot[kk] += v
            tot["flops"] += 2.0 * m * n * k
        fl = tot.pop("flops")
        res[f"subgrid_2^7..2^11_threads={threads}"] = {
            **{f"{kk}_tflops": fl / v / 1e12 for kk, v in tot.items()},
            "port_over_ref_nt": tot["ref_nt"] / tot["port_nt"],
            "port_over_ref_tnn": tot["ref_tnn"] / tot["port_tnn"],
        }
    Path(out_path).parent.mkdir(parents=True, exist_ok=True)
    Path(out_path).write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
