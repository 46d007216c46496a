"""B200 timing sweep: NN, NT and TNN per (m, n, k) case, for labeling and retraining.

GPU restatement of the reference harness (/root/reference/pkg/src/mtnn/bench.py):
``grid_shapes`` (:198-205, 2^e per dimension, lexicographic), ``make_operands``
semantics (:104-114, uniform [-1, 1]), interleaved round-robin timing with warm-up
and median (:129-146), and the timings CSV wire format ``m,n,k,t_nn,t_nt,t_tnn``
(:36-38, :366-363) that the reference's fixture mode reads back
(``read_timings_csv`` -> ``sweep_grid(injected=...)`` -> ``label_records`` ->
``fit_gbdt``), so the reference learner retrains unchanged on B200 labels.

Timing: CUDA events on the launching stream around each call, an L2 flush
(a 256 MiB read, > the 126 MB L2, leaving no dirty lines to write back) and a
short GPU spin (so the host's enqueue gaps stay outside the window) before every
timed call, inputs resident in HBM. TNN's window includes its stream-ordered B^T allocation, transpose and
release (reference _numba_impl.py:16-19); the NN time uses a
pre-transposed B^T, as the reference's does (bench.py:208-229).
"""

from __future__ import annotations

import csv
import itertools
import statistics
from dataclasses import dataclass

import torch

from . import _lib
from . import device

TIMING_HEADER = ("m", "n", "k", "t_nn", "t_nt", "t_tnn")
# wire contracts shared with the reference learner (bench.py:34-38)
SAMPLE_HEADER = ("gm", "sm", "cc", "mbw", "l2c", "m", "n", "k", "label")
RECORD_HEADER = ("m", "n", "k", "p_nn", "p_nt", "p_tnn", "t_nt", "t_tnn")


def grid_shapes(exponents):
    sizes = [2 ** e for e in exponents]
    return list(itertools.product(sizes, sizes, sizes))


class Operands:
    """Max-size resident operands; each case views a prefix (synthetic data)."""

    def __init__(self, max_m, max_n, max_k, seed=0, dev="cuda"):
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        self.a = torch.rand(max_m * max_k, device=dev, generator=g).mul_(2).sub_(1)
        self.b = torch.rand(max_n * max_k, device=dev, generator=g).mul_(2).sub_(1)
        self.bt = torch.empty(max_n * max_k, device=dev)
        self.c = torch.empty(max_m * max_n, device=dev)
        self.flush_buf = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def views(self, m, n, k):
        a = self.a[: m * k].view(m, k)
        b = self.b[: n * k].view(n, k)
        c = self.c[: m * n].view(m, n)
        return a, b, c

    def flush(self):
        self.flush_buf.sum()
        torch.cuda._sleep(200_000)


def time_calls(fns: dict, ops: Operands, reps: int, warmup: int) -> dict:
    """Per-name median seconds, round-robin interleaved, L2 flushed before each."""
    for _ in range(warmup):
        for fn in fns.values():
            fn()
    events = {name: [] for name in fns}
    for _ in range(reps):
        for name, fn in fns.items():
            ops.flush()
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            events[name].append((s, e))
    torch.cuda.synchronize()
    return {name: statistics.median(s.elapsed_time(e) * 1e-3 for s, e in evs)
            for name, evs in events.items()}


@dataclass
class CaseTiming:
    m: int
    n: int
    k: int
    t_nn: float
    t_nt: float
    t_tnn: float


def measure_case(ops: Operands, m, n, k, reps=5, warmup=2, variant=_lib.VARIANT_AUTO):
    a, b, c = ops.views(m, n, k)
    bt = ops.bt[: n * k].view(k, n)
    device.transpose(b, out=bt)
    fns = {
        "nn": lambda: device.gemm_nn(a, bt, out=c, variant=variant),
        "nt": lambda: device.gemm_nt(a, b, out=c, variant=variant),
        "tnn": lambda: device.gemm_tnn(a, b, out=c, variant=variant),
    }
    t = time_calls(fns, ops, reps, warmup)
    return CaseTiming(m, n, k, t["nn"], t["nt"], t["tnn"])


def sweep_shapes(shapes, reps=5, warmup=2, variant=_lib.VARIANT_AUTO, log=None):
    """CaseTiming per (m, n, k) of `shapes`, in order, on the current device."""
    shapes = [tuple(int(v) for v in s) for s in shapes]
    if not shapes:
        return []
    ops = Operands(max(s[0] for s in shapes), max(s[1] for s in shapes),
                   max(s[2] for s in shapes))
    out = []
    for (m, n, k) in shapes:
        ct = measure_case(ops, m, n, k, reps, warmup, variant)
        out.append(ct)
        if log:
            log(f"{m} {n} {k}: nn {ct.t_nn*1e6:.1f}us nt {ct.t_nt*1e6:.1f}us "
                f"tnn {ct.t_tnn*1e6:.1f}us  NT {2*m*n*k/ct.t_nt/1e12:.1f} TF")
    return out


def sweep(exponents, reps=5, warmup=2, variant=_lib.VARIANT_AUTO, log=None, gpus=1, first=0):
    """The grid sweep; gpus > 1 shards the cases over GPUs first..first+gpus-1."""
    shapes = grid_shapes(exponents)
    if gpus > 1:
        return map_cases_on_gpus(_sweep_worker, shapes, gpus, (reps, warmup, variant), first)
    return sweep_shapes(shapes, reps, warmup, variant, log)


# --------------------------------------------------------- multi-GPU cases
def lpt_shards(shapes, parts):
    """Longest-processing-time-first assignment of cases (cost 2mnk) to parts."""
    loads = [0.0] * parts
    owner = [0] * len(shapes)
    for i in sorted(range(len(shapes)), key=lambda j: -(shapes[j][0] * shapes[j][1] * shapes[j][2])):
        r = min(range(parts), key=lambda q: loads[q])
        owner[i] = r
        loads[r] += float(shapes[i][0]) * shapes[i][1] * shapes[i][2]
    return owner


def _sweep_worker(dev, shapes, extra):
    torch.cuda.set_device(dev)
    return sweep_shapes(shapes, *extra)


def _pool_entry(fn, slot_dev, shapes, extra, q):
    try:
        q.put((slot_dev, fn(slot_dev[1], shapes, extra), None))
    except BaseException as exc:  # noqa: BLE001 - reported to the parent
        q.put((slot_dev, None, f"{type(exc).__name__}: {exc}"))


def map_cases_on_gpus(fn, shapes, gpus, extra, first=0, devices=None):
    """Run fn(device, shapes_part, extra) -> list (one result per shape) in one
    process per GPU (spawned; cases LPT-sharded, no collective) and return the
    results in the order of `shapes`. Independent cases need no exchange.
    `devices` (tests) overrides the device list first..first+gpus-1."""
    import multiprocessing as mp

    if devices is None:
        have = torch.cuda.device_count()
        if first < 0 or first + gpus > have:
            raise ValueError(f"GPUs {first}..{first + gpus - 1} requested but {have} CUDA devices "
                             f"are visible")
        devices = list(range(first, first + gpus))
    owner = lpt_shards([tuple(s) for s in shapes], len(devices))
    parts = [[s for s, o in zip(shapes, owner) if o == d] for d in range(len(devices))]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pool_entry, args=(fn, (slot, dev), parts[slot], extra, q))
             for slot, dev in enumerate(devices)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        (slot, dev), res, err = q.get()
        if err is not None:
            for p in procs:
                p.join(timeout=5)
            raise RuntimeError(f"GPU {dev}: {err}")
        got[slot] = iter(res)
    for p in procs:
        p.join()
    return [next(got[o]) for o in owner]


def write_timings_csv(path, rows):
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(TIMING_HEADER)
        for r in rows:
            w.writerow([r.m, r.n, r.k, repr(r.t_nn), repr(r.t_nt), repr(r.t_tnn)])


def gflops(m, n, k, seconds):
    if not seconds > 0:
        raise ValueError(f"duration must be positive, got {seconds}")
    return 2.0 * m * n * k / (seconds * 1e9)


def record_of(r: CaseTiming) -> tuple:
    """(m, n, k, p_nn, p_nt, p_tnn, t_nt, t_tnn) — the reference BenchRecord row."""
    return (r.m, r.n, r.k, gflops(r.m, r.n, r.k, r.t_nn), gflops(r.m, r.n, r.k, r.t_nt),
            gflops(r.m, r.n, r.k, r.t_tnn), r.t_nt, r.t_tnn)


def label_of(r: CaseTiming) -> int:
    """+1 (NT) iff p_nt - p_tnn >= 0, else -1 (TNN) — reference bench.py:296-303."""
    rec = record_of(r)
    return 1 if rec[4] - rec[5] >= 0 else -1


def write_records_csv(path, rows):
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(RECORD_HEADER)
        for r in rows:
            w.writerow(list(record_of(r)))


def write_samples_csv(path, rows, platform):
    """Training samples (5 platform features + m, n, k, label), floats as repr."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(SAMPLE_HEADER)
        for r in rows:
            feats = tuple(platform.as_tuple()) + (float(r.m), float(r.n), float(r.k))
            w.writerow([repr(float(v)) for v in feats] + [label_of(r)])


def rows_from_timings(timings: dict) -> list:
    """CaseTiming rows from {(m, n, k): (t_nn, t_nt, t_tnn)} (injected timings)."""
    return [CaseTiming(m, n, k, *t) for (m, n, k), t in timings.items()]


def read_timings_csv(path):
    out = {}
    with open(path, newline="") as fh:
        rd = csv.DictReader(fh)
        for row in rd:
            out[(int(row["m"]), int(row["n"]), int(row["k"]))] = (
                float(row["t_nn"]), float(row["t_nt"]), float(row["t_tnn"]))
    return out


if __name__ == "__main__":
    import argparse
    import json
    import sys

    from .platform import probe_platform

    ap = argparse.ArgumentParser(description="B200 NN/NT/TNN timing sweep")
    ap.add_argument("--exp-min", type=int, default=7)
    ap.add_argument("--exp-max", type=int, default=14)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--variant", default="auto", choices=sorted(_lib.VARIANTS))
    ap.add_argument("--out", default="gpurun_out/sweep_timings.csv")
    args = ap.parse_args()
    rows = sweep(range(args.exp_min, args.exp_max + 1), args.reps, args.warmup,
                 _lib.VARIANTS[args.variant], log=lambda s: print(s, file=sys.stderr, flush=True))
    write_timings_csv(args.out, rows)
    plat = probe_platform()
    with open(args.out + ".platform.json", "w") as fh:
        json.dump({"platform": plat.as_tuple(), "variant": args.variant,
                   "reps": args.reps, "warmup": args.warmup}, fh)
    print(f"wrote {len(rows)} cases to {args.out}")
