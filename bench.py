"""MTNN B200 benchmark — BASELINE.json's metric on its sweep configuration.

Workload (configs[1]): the NT sweep m, n, k in {128, ..., 16384} (512 cases),
every case computed C = A B^T through the MTNN dispatcher (GBDT decision in
host C++, then the direct-NT or the TNN path on sm_100a), on the reference
harness's operands make_operands(shape, seed 0) (bench.py:104-114; generated
on the device bit-identically, every case a view of one seed-0 stream). One
"step" = one pass over all cases. `value` = total flops / total device time
(whole job), inputs resident in HBM, L2 flushed (256 MiB read) before every
case and excluded from the timed windows. After the timed steps the bench
checks its own outputs (a sampled block of every case against float64) and
times MTNN, NT and TNN per case interleaved in one pass (MTNN vs the per-case
best of both). `e2e` = the same sweep through the reference-facing C-ABI with
pinned HOST buffers (H2D of A and B, D2H of C inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload sweep|single|fcn|large]

N > 1 (torchrun, one rank per GPU, NCCL): sweep cases are assigned to ranks
longest-first (no collective); `large` row-shards A with B broadcast and the
all-gather of C fused into the GEMM epilogue; `fcn` is data parallel with an
all-reduce of the weight gradients. `--impl reference` times the reference's
CPU implementation of the path (the reference itself from baseline/_ref when it
is installed, else the C restatement in oracle/; all host threads) on a bounded
sample of the same workload and reports the same `config`.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SLEEP_CYCLES = 200_000  # ~0.1 ms at 1.9 GHz of GPU spin ahead of each timed window
METRIC = "NT A·Bᵀ TFLOPS (MTNN-selected) over m,n,k sweep; transpose GB/s; selector accuracy"
DEFAULT_MODEL = ROOT / "paper_1702_03192_b200" / "models" / "b200_sweep.json"


def grid(exp_min, exp_max):
    s = [2 ** e for e in range(exp_min, exp_max + 1)]
    return [(m, n, k) for m in s for n in s for k in s]


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:7], float(parts[7])))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [r for r in rows if r[3] > 0] or rows
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(loaded)}


class NvmlClockSampler:
    """NVML sampled every 2 ms during the timed region (short workloads — the FCN
    step is ~1 ms — finish between nvidia-smi samples); ClockSampler otherwise."""

    # NVML clocks-event-reason bits: sw power cap, hw slowdown, sw / hw thermal
    BITS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
            ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        import pynvml

        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        self.rows = []
        self.stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                util = float(nv.nvmlDeviceGetUtilizationRates(self.h).gpu)
                self.rows.append((mhz, bits, util))
            except Exception:  # noqa: BLE001  (a failed sample is skipped)
                pass
            self.stop.wait(0.002)

    def __enter__(self):
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        self.thread.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        loaded = [r for r in self.rows if r[2] > 0] or self.rows
        reasons = sorted({name for r in loaded for name, bit in self.BITS if r[1] & bit})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "samples_under_load": len(loaded),
                "sampler": "nvml 2 ms"}


def clock_sampler(index: int):
    try:
        return NvmlClockSampler(index)
    except Exception:  # noqa: BLE001  (no NVML: nvidia-smi at 100 ms)
        return ClockSampler(index)


# ----------------------------------------------------------------- CPU legs
class CpuRef:
    """The reference's CPU kernels for the CPU legs. Preferred: the reference
    itself (baseline/_ref, installed unmodified by tools/install_reference.sh;
    numba backend, its public kernels API: kernels.gemm_nt / gemm_nn /
    transpose_oop / gemm_tnn with threads=) — kind "reference". Fallback when
    it is absent or numba is not importable: the oracle/ C port of the same
    loops — kind "port" (measured 0.97x the reference on NT and 0.69x on TNN
    at 16 threads, profiles/ref_vs_port_r02.json). MTNN_BENCH_CPU=port forces
    the port."""

    def __init__(self):
        self.kind, self.label = "port", "oracle/ C port of the reference numba kernels"
        self._k = None
        ref = ROOT / "baseline" / "_ref"
        if os.environ.get("MTNN_BENCH_CPU") != "port" and (ref / "mtnn").is_dir():
            try:
                os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mtnn_bench_numba")
                os.environ["MTNN_BACKEND"] = "numba"
                sys.path.insert(0, str(ref))
                from mtnn import kernels as rk  # noqa: WPS433  (the unmodified reference)

                if rk.active_backend() == "numba":
                    self._k, self.kind = rk, "reference"
                    self.label = "the reference (baseline/_ref, numba backend, mtnn.kernels API)"
            except Exception as exc:  # noqa: BLE001 - fall back to the port, say why
                self.label += f" (reference unavailable: {type(exc).__name__})"
        if self._k is None:
            import oracle

            self._o = oracle

    def gemm_nt(self, a, b, threads):
        return (self._k.gemm_nt(a, b, threads=threads) if self._k else
                self._o.gemm_nt(a, b, threads=threads))

    def gemm_nn(self, a, bt, threads):
        return (self._k.gemm_nn(a, bt, threads=threads) if self._k else
                self._o.gemm_nn(a, bt, threads=threads))

    def transpose(self, b):  # single-threaded in both (the reference has no parallel transpose)
        return self._k.transpose_oop(b) if self._k else self._o.transpose(b, threads=1)

    def gemm_tnn(self, a, b, threads):
        return (self._k.gemm_tnn(a, b, threads=threads) if self._k else
                self._o.gemm_tnn(a, b, threads=threads))

    def warm(self, threads):
        """JIT-compile / page in every kernel and thread-pool once (untimed)."""
        rng = np.random.default_rng(1)
        a = rng.uniform(-1, 1, (64, 48)).astype(np.float32)
        b = rng.uniform(-1, 1, (40, 48)).astype(np.float32)
        for t in sorted({1, threads}):
            self.gemm_nt(a, b, t)
            self.gemm_nn(a, np.ascontiguousarray(b.T), t)
            self.gemm_tnn(a, b, t)
        self.transpose(b)


_CPU = None


def cpu_ref():
    global _CPU
    if _CPU is None:
        _CPU = CpuRef()
    return _CPU


CPU_ROW_FLOP_CAP = 2 ** 28
CPU_MIN_ROWS = 16


def cpu_rows(m, n, k):
    return min(m, max(CPU_MIN_ROWS, CPU_ROW_FLOP_CAP // (2 * n * k)))


def cpu_sweep_sample(shapes, threads):
    """(flops, seconds best-of-both, seconds NT, seconds TNN) extrapolated from
    row samples of `shapes`; operands are uniform[-1,1) (timing does not depend
    on the values)."""
    ref = cpu_ref()
    n_max = max(n for _, n, _ in shapes)
    k_max = max(k for _, _, k in shapes)
    rng = np.random.default_rng(0)
    b_buf = rng.uniform(-1, 1, n_max * k_max).astype(np.float32)
    a_buf = rng.uniform(-1, 1, max(cpu_rows(m, n, k) * k for m, n, k in shapes)).astype(np.float32)
    by_nk = {}
    for (m, n, k) in shapes:
        by_nk.setdefault((n, k), []).append(m)
    flops = s_best = s_nt = s_tnn = 0.0
    for (n, k), ms in by_nk.items():
        b = b_buf[: n * k].reshape(n, k)
        t0 = time.perf_counter()
        bt = ref.transpose(b)
        t_tr = time.perf_counter() - t0
        for m in ms:
            r = cpu_rows(m, n, k)
            a = a_buf[: r * k].reshape(r, k)
            t0 = time.perf_counter()
            ref.gemm_nt(a, b, threads)
            t1 = time.perf_counter()
            ref.gemm_nn(a, bt, threads)
            t2 = time.perf_counter()
            t_nt = (t1 - t0) * m / r
            t_tnn = t_tr + (t2 - t1) * m / r
            flops += 2.0 * m * n * k
            s_nt += t_nt
            s_tnn += t_tnn
            s_best += min(t_nt, t_tnn)
    return flops, s_best, s_nt, s_tnn


def cpu_single(m, n, k, threads, seed=0):
    """configs[0]: the full NT op through both reference paths on make_operands."""
    ref = cpu_ref()
    rng = np.random.default_rng(seed)  # make_operands (reference bench.py:104-114)
    a = rng.uniform(-1.0, 1.0, (m, k)).astype(np.float32)
    b = rng.uniform(-1.0, 1.0, (n, k)).astype(np.float32)
    t0 = time.perf_counter()
    ref.gemm_nt(a, b, threads)
    t1 = time.perf_counter()
    ref.gemm_tnn(a, b, threads)
    t2 = time.perf_counter()
    return 2.0 * m * n * k, min(t1 - t0, t2 - t1), t1 - t0, t2 - t1


def cpu_sample_text(args, threads, per_step=False):
    if args.workload == "single":
        return (f"the full {args.single}^3 NT op (make_operands seed 0), {cpu_ref().label}, "
                f"faster of NT / TNN, {threads} threads")
    if args.workload == "fcn":
        return (f"the full FCN step (12 products), {cpu_ref().label}, NT products: faster of "
                f"NT / TNN, {threads} threads")
    if per_step:
        return (f"each step: every {CPU_PARTS}th case of the sweep (offset by the step; "
                f"{CPU_PARTS} steps cover all {len(grid(args.exp_min, args.exp_max))}), "
                + cpu_sample_text(args, threads).split(", ", 1)[1])
    return (f"all {len(grid(args.exp_min, args.exp_max))} cases of the sweep, each on its first "
            f"min(m, max({CPU_MIN_ROWS}, 2^28 flop / 2nk)) rows of A at full n, k, time scaled by "
            f"m / rows (both reference paths are per-row linear; TNN adds its full single-thread "
            f"transpose of B per (n, k)); {cpu_ref().label}, faster "
            f"of NT / TNN per case, {threads} threads")


CPU_PARTS = 4  # reference-arm steps rotate over quarters of the sweep's cases


def cpu_part(args, step):
    """Cases of reference-arm step `step`: every CPU_PARTS-th case of the grid,
    offset by the step, so CPU_PARTS consecutive steps cover the whole sweep."""
    return grid(args.exp_min, args.exp_max)[step % CPU_PARTS::CPU_PARTS]


def cpu_run(args, threads, step=None):
    """(flops, s_best, s_nt, s_tnn): the whole workload (step None) or one
    reference-arm step's part of it."""
    if args.workload == "single":
        n = args.single
        return cpu_single(n, n, n, threads)
    if args.workload == "fcn":
        return cpu_fcn(threads)
    shapes = grid(args.exp_min, args.exp_max) if step is None else cpu_part(args, step)
    return cpu_sweep_sample(shapes, threads)


def cpu_fcn(threads):
    """configs[3] on the CPU reference: the FCN step's 12 products at full size
    (forward NT and backward weight-gradient NT: faster of the two reference
    paths; backward NN: the blocked NN kernel)."""
    ref = cpu_ref()
    rng = np.random.default_rng(0)
    widths = list(FCN_LAYERS)
    layers = list(zip(widths[:-1], widths[1:]))
    calls = [("nt", FCN_BATCH, dout, din) for din, dout in layers]
    for din, dout in reversed(layers):
        calls += [("nn", FCN_BATCH, din, dout), ("nt", dout, din, FCN_BATCH)]
    flops = s_best = s_nt = s_tnn = 0.0
    for op, m, n, k in calls:
        a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        b = rng.uniform(-1, 1, (k, n) if op == "nn" else (n, k)).astype(np.float32)
        flops += 2.0 * m * n * k
        if op == "nn":
            t0 = time.perf_counter()
            ref.gemm_nn(a, b, threads)
            t = time.perf_counter() - t0
            s_best += t
            s_nt += t
            s_tnn += t
            continue
        t0 = time.perf_counter()
        ref.gemm_nt(a, b, threads)
        t1 = time.perf_counter()
        ref.gemm_tnn(a, b, threads)
        t2 = time.perf_counter()
        s_nt += t1 - t0
        s_tnn += t2 - t1
        s_best += min(t1 - t0, t2 - t1)
    return flops, s_best, s_nt, s_tnn


def host_threads() -> int:
    """All host cores this process may run on (torchrun sets OMP_NUM_THREADS=1,
    so the OpenMP default is not the machine's core count)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(args, threads: int):
    cpu_ref().warm(threads)
    flops, best, s_nt, s_tnn = cpu_run(args, threads)
    return {
        "value": flops / best / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": cpu_ref().kind,
        "sample": cpu_sample_text(args, threads)
                  + f"; always-NT {flops / s_nt / 1e12:.4f}, always-TNN {flops / s_tnn / 1e12:.4f} TFLOP/s",
        "seconds": best,
    }


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path (CpuRef:
    the reference itself, else the oracle port), timed on the host cores, rank 0 only, on the same workload/config as
    the GPU arm (a bounded sample of it; see cpu_sweep_sample)."""
    if rank != 0:
        return
    if args.workload == "large":
        print(json.dumps({"impl": "reference", "unavailable":
                          "configs[4] (65536x8192x8192) is ~9e12 flop, about a minute of CPU work "
                          "per step even on every host core; the sweep/single/fcn arms cover the "
                          "CPU reference"}), flush=True)
        return
    threads = host_threads()
    cpu_ref().warm(threads)
    for _ in range(args.warmup):  # warm caches / the thread pool on a few cases
        if args.workload == "sweep":
            cpu_sweep_sample(grid(args.exp_min, min(args.exp_max, args.exp_min + 2)), threads)
        else:
            cpu_single(256, 256, 256, threads)
    est, walls, flops = [], [], 0.0
    for step in range(args.steps):
        t0 = time.perf_counter()
        f, best, _, _ = cpu_run(args, threads, step)
        walls.append(time.perf_counter() - t0)
        est.append(best)
        flops += f
    # whole-job throughput: flops of the cases the steps covered / their
    # (row-sample extrapolated) CPU time
    value = flops / sum(est) / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(walls) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, world, workload_desc(args, world)),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads,
                         "kind": cpu_ref().kind,
                         "sample": cpu_sample_text(args, threads, per_step=True),
                         "cpu_seconds_per_step_of_the_covered_cases": statistics.mean(est)},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- workloads
def lpt_assign(costs, world):
    """Longest-processing-time-first assignment of independent cases to ranks."""
    loads = [0.0] * world
    owner = [0] * len(costs)
    for i in sorted(range(len(costs)), key=lambda j: -costs[j]):
        r = min(range(world), key=lambda q: loads[q])
        owner[i] = r
        loads[r] += costs[i]
    return owner


FCN_LAYERS = (784, 4096, 4096, 4096, 10)
FCN_BATCH = 1024
LARGE = (65536, 8192, 8192)


def model_name_of(args):
    return Path(args.model).name if Path(args.model).exists() else "empty (always NT)"


def workload_desc(args, world):
    """(workload description, parallelism) — shared by both arms' `config`."""
    if args.workload == "sweep":
        n = len(grid(args.exp_min, args.exp_max))
        desc = (f"nt_sweep m,n,k in {{2^{args.exp_min}..2^{args.exp_max}}} ({n} cases), "
                f"MTNN-selected (configs[1])")
        par = "single GPU" if world == 1 else f"cases LPT-sharded over {world} GPUs (no collective)"
        return desc, par
    if args.workload == "single":
        s = args.single
        return (f"single NT op m=n=k={s} through the MTNN dispatcher (configs[0])",
                "single GPU" if world == 1 else f"{world} independent replicas")
    if args.workload == "fcn":
        desc = ("fcn_step 784-4096-4096-4096-10 batch 1024 (configs[3]): 4 forward NT + 4 backward "
                "NN + 4 backward NT, all NT through MTNN (the reference routes only forward NT)")
        par = ("single GPU" if world == 1 else
               f"data parallel x{world}: batch 1024 per GPU, weight gradients all-reduced (NCCL, "
               f"overlapped with the remaining backward GEMMs)")
        return desc, par
    desc = "large_nt m=65536 n=k=8192 (configs[4]), rows of A sharded, B replicated"
    par = ("single GPU" if world == 1 else
           f"row-sharded x{world}: NCCL broadcast of B, then the all-gather of C "
           + ("fused into the GEMM epilogue (peer stores over NVLink) with device-side barriers"
              if args.gather == "fused" else "by ncclAllGather"))
    return desc, par


def workload_config(args, world, desc_par):
    desc, par = desc_par
    cfg = {"workload": desc, "model": model_name_of(args),
           "operands": ("make_operands(shape, seed 0) (reference bench.py:104-114)"
                        if args.workload in ("sweep", "single", "large") else
                        "uniform[-1,1) activations/weights (seeded torch generator)"),
           "l2": "flushed (256 MiB read) before every case/phase, outside the timed windows",
           "parallelism": par,
           "precision": ("FP32-accurate: 3 tensor-core MMAs per product on hi/lo operand "
                         "halves (pow2-scaled FP16, or TF32) with FP32 promotion, or FP32 FFMA")}
    if args.workload == "sweep":
        cfg["cases"] = len(grid(args.exp_min, args.exp_max))
    return cfg


def build_workload(args, rank, world):
    """Per-step call list for this rank: (op, m, n, k, flush_before).
    op: "nt" = MTNN-dispatched NT, "nn" = NN product, "grad" = an FCN weight-gradient
    NT (MTNN-dispatched into its own buffer; all-reduced across ranks when N > 1)."""
    if args.workload == "sweep":
        shapes = grid(args.exp_min, args.exp_max)
        owner = lpt_assign([2.0 * m * n * k for m, n, k in shapes], world)
        calls = [("nt", m, n, k, True) for (m, n, k), o in zip(shapes, owner) if o == rank]
        total = sum(2.0 * m * n * k for m, n, k in shapes)
        return calls, total, "strong", shapes
    if args.workload == "single":
        s = args.single
        return [("nt", s, s, s, True)], 2.0 * s ** 3 * world, ("weak" if world > 1 else "strong"), \
            [(s, s, s)]
    if args.workload == "fcn":
        widths = list(FCN_LAYERS)
        layers = list(zip(widths[:-1], widths[1:]))
        calls = [("nt", FCN_BATCH, dout, din, i == 0) for i, (din, dout) in enumerate(layers)]
        for j, (din, dout) in enumerate(reversed(layers)):
            calls.append(("nn", FCN_BATCH, din, dout, j == 0))
            calls.append(("grad", dout, din, FCN_BATCH, False))  # weight gradient (an NT)
        total = sum(2.0 * m * n * k for _, m, n, k, _ in calls) * world
        return calls, total, ("weak" if world > 1 else "strong"), None
    # large (config 5): m = 65536 rows of A sharded, B replicated
    from paper_1702_03192_b200.sharding import row_range

    m, n, k = LARGE
    lo, hi = row_range(m, rank, world)
    return [("nt", hi - lo, n, k, True)], 2.0 * m * n * k, "strong", None


# ----------------------------------------------------------------- GPU legs
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="sweep", choices=("sweep", "single", "fcn", "large"))
    ap.add_argument("--single", type=int, default=1024,
                    help="single workload (configs[0]): m = n = k")
    ap.add_argument("--oracle-reps", type=int, default=5,
                    help="sweep: reps of the interleaved MTNN / NT / TNN per-case pass")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--exp-min", type=int, default=7)
    ap.add_argument("--exp-max", type=int, default=14)
    ap.add_argument("--model", default=str(DEFAULT_MODEL))
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--gather", default="fused", choices=("fused", "nccl"),
                    help="large workload, N > 1: all-gather of C fused into the GEMM epilogue "
                         "(peer stores over CUDA IPC / NVLink) or an ncclAllGather after it")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import ctypes

    import torch
    import torch.distributed as dist

    # one rank per GPU; MTNN_BENCH_SHARE_GPU=1 maps ranks onto the visible GPUs
    # modulo their count and uses gloo (test mode for the N>1 path on one GPU)
    share = os.environ.get("MTNN_BENCH_SHARE_GPU") == "1"
    local_rank = local_rank % torch.cuda.device_count() if share else local_rank
    torch.cuda.set_device(local_rank)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    from paper_1702_03192_b200 import ProblemShape, _lib, gbdt
    from paper_1702_03192_b200.platform import probe_platform
    from paper_1702_03192_b200.selector import Dispatcher

    dev = torch.device("cuda", local_rank)
    L = _lib.lib
    calls, total_flops, scaling, shapes = build_workload(args, rank, world)
    desc_par = workload_desc(args, world)

    # model: the B200-trained selector if present, else an empty model (always NT)
    if Path(args.model).exists():
        model = gbdt.load_model(args.model)
    else:
        model = gbdt.GbdtModel(trees=(), params=gbdt.GbdtParams(), n_features=8)
    disp = Dispatcher(model, probe_platform())
    handle = disp._native.handle
    prefix_p = disp._prefix_p

    # resident operands. sweep/single/large: the reference harness's
    # make_operands(shape, 0) — A = draws [0, m k) of seed 0, B = the next n k —
    # so one seed-0 stream on the device holds every case's A and B as views.
    # fcn: seeded uniform activations / weights (the reference's fcn builds its own).
    from paper_1702_03192_b200 import operands as _ops

    cap_c = max([m * n for _, m, n, k, _ in calls] + [1])
    if args.workload == "large":
        cap_c = LARGE[0] * LARGE[1]  # gathered C
    if args.workload == "fcn":
        g = torch.Generator(device=dev)
        g.manual_seed(1234 + rank)
        A = torch.rand(max(m * k for _, m, n, k, _ in calls), device=dev, generator=g).mul_(2).sub_(1)
        B = torch.rand(max(n * k for _, m, n, k, _ in calls), device=dev, generator=g).mul_(2).sub_(1)
        ab_ptrs = [(A.data_ptr(), B.data_ptr()) for _ in calls]
        a_views = [A[: m * k].view(m, k) for _, m, n, k, _ in calls]
        b_views = [B[: n * k].view(k, n) if op == "nn" else B[: n * k].view(n, k)
                   for op, m, n, k, _ in calls]
    elif args.workload == "large":
        from paper_1702_03192_b200.sharding import row_range

        M, N, K = LARGE
        A = _ops.operand_stream(M * K + N * K, seed=0, device=dev)
        lo, hi = row_range(M, rank, world)
        B = A[M * K:]
        a_views = [A[lo * K: hi * K].view(hi - lo, K)]
        b_views = [B.view(N, K)]
        ab_ptrs = [(a_views[0].data_ptr(), B.data_ptr())]
    else:
        A = _ops.operand_stream(max(m * k + n * k for _, m, n, k, _ in calls), seed=0, device=dev)
        B = A
        a_views = [A[: m * k].view(m, k) for _, m, n, k, _ in calls]
        b_views = [A[m * k: m * k + n * k].view(n, k) for _, m, n, k, _ in calls]
        ab_ptrs = [(A.data_ptr(), A.data_ptr() + 4 * m * k) for _, m, n, k, _ in calls]
    C = torch.empty(cap_c, device=dev)
    # L2 flush by READING 256 MiB (> 126 MB L2): leaves clean lines, so the next
    # timed kernel does not pay the write-back of a dirty flush buffer
    flush_src = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    choice = ctypes.c_int()

    # FCN weight gradients get their own buffers (all-reduced across ranks while
    # later backward GEMMs run)
    grad_bufs = {}
    if args.workload == "fcn":
        for i, (op, m, n, k, _) in enumerate(calls):
            if op == "grad":
                grad_bufs[i] = torch.empty(m * n, device=dev)

    # large workload, N > 1, fused gather: every rank's full C is mapped by the
    # others (CUDA IPC) and the GEMM epilogue stores each tile into all of them
    peer_gather, gather_mode = None, None
    if args.workload == "large" and world > 1:
        gather_mode = args.gather
        if args.gather == "fused":
            from paper_1702_03192_b200.sharding import PeerGather

            try:
                peer_gather = PeerGather(C[: LARGE[0] * LARGE[1]].view(LARGE[0], LARGE[1]))
                large_row0 = lo
            except Exception as exc:  # no IPC between these processes: NCCL fallback
                gather_mode = f"nccl (fused unavailable: {type(exc).__name__}: {exc})"[:200]
                peer_gather = None

    def run_call(i, out=None):
        op, m, n, k, _ = calls[i]
        if m <= 0:
            return
        if peer_gather is not None:
            peer_gather.gemm(a_views[i], b_views[i], large_row0, sync=False)
            return
        pa, pb = ab_ptrs[i]
        if op == "grad":
            rc = L.mtnn_dispatch_gemm(handle, prefix_p, pa, pb, out.data_ptr(),
                                      m, n, k, -1, 0, stream, ctypes.byref(choice))
        elif op == "nt":
            rc = L.mtnn_dispatch_gemm(handle, prefix_p, pa, pb, C.data_ptr(),
                                      m, n, k, -1, 0, stream, ctypes.byref(choice))
        else:
            rc = L.mtnn_gemm_nn(pa, pb, C.data_ptr(), m, n, k, 0, stream)
        if rc:
            _lib.check(rc)

    def out_view(i):
        op, m, n, k, _ = calls[i]
        if op == "grad":
            return grad_bufs[i][: m * n].view(m, n)
        if peer_gather is not None:
            return C[large_row0 * n: (large_row0 + m) * n].view(m, n)
        return C[: m * n].view(m, n)

    comm = {"bcast": [], "gather": [], "allreduce": []}
    gate_t = torch.zeros(1, dtype=torch.int32).pin_memory()  # mtnn_gate release flag
    gate_np, gate_ptr, gate_seq = gate_t.numpy(), gate_t.data_ptr(), [0]
    # under a profiler (ncu serialises kernels: the host could never release a
    # held gate, each would wait out its 1 s bound) fall back to the GPU spin;
    # no number taken under a profiler is a bench value anyway
    use_gate = (os.environ.get("MTNN_BENCH_GATE", "1") != "0"
                and not any(k in os.environ for k in ("CUDA_INJECTION64_PATH", "NV_COMPUTE_PROFILER_PERFWORKS_DIR")))

    from paper_1702_03192_b200.sharding import allreduce_weight_grad as allreduce_grad

    def one_step(events=None):
        if args.workload == "large" and world > 1:
            # B replicated from rank 0, timed as part of the sharded op
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
            dist.broadcast(B[: LARGE[1] * LARGE[2]], src=0)
            ev[1].record()
            if events is not None:
                comm["bcast"].append(ev)
                events.append(ev)
        works = []
        for i, (op, m, n, k, fl) in enumerate(calls):
            if fl:
                flush_src.sum()
            if events is not None and not use_gate:
                torch.cuda._sleep(SLEEP_CYCLES)
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                s.record()
                run_call(i, grad_bufs.get(i))
                e.record()
                events.append((s, e))
            elif events is not None:
                # hold the stream at a gate until the whole call is enqueued, so
                # the event window holds device work only: a host stall while
                # enqueueing (GIL, page fault) would otherwise sit inside the
                # open window as GPU idle time (tools/probes/probe_outliers.py).
                # The warm-up steps have loaded every kernel and grown the pools
                # (a lazy module load behind a held gate would synchronise).
                gate_seq[0] += 1
                _lib.check(L.mtnn_gate(gate_ptr, gate_seq[0], stream))
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                s.record()
                run_call(i, grad_bufs.get(i))
                e.record()
                gate_np[0] = gate_seq[0]  # release
                events.append((s, e))
            else:
                torch.cuda._sleep(SLEEP_CYCLES)
                run_call(i, grad_bufs.get(i))
            if op == "grad" and world > 1:
                works.append(allreduce_grad(grad_bufs[i]))
        if args.workload == "fcn" and world > 1:
            # the all-reduces still in flight after the last GEMM: their tail is
            # part of the step
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
            for w in works:
                if w is not None:
                    w.wait()
            ev[1].record()
            if events is not None:
                comm["allreduce"].append(ev)
                events.append(ev)
        if args.workload == "large" and world > 1 and peer_gather is None:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
            rows = calls[0][1]
            if dist.get_backend() == "nccl":
                dist.all_gather_into_tensor(C[: 65536 * 8192], C[: rows * 8192].clone())
            else:  # gloo test mode (equal row blocks)
                dist.all_gather(list(C[: 65536 * 8192].chunk(world)), C[: rows * 8192].clone())
            ev[1].record()
            if events is not None:
                comm["gather"].append(ev)
                events.append(ev)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()

    # ---------------- timed region: K steps
    # Only the large GEMM launches carry timing events here (the roofline kernel,
    # calls of >= 2^35 flop, or the largest call if none is that big): a
    # timestamp event pair serialises the stream around its launch and breaks
    # the programmatic launch chain, which costs ~4% of a sweep step when every
    # launch is bracketed (3% with every GEMM bracketed). All launches are still
    # counted. The per-class breakdown comes from one extra fully instrumented
    # step after the timed region.
    min_work = min(float(2 ** 35), max((2.0 * m * n * k for _, m, n, k, _ in calls), default=0.0))
    # a step of several mid-size launches at that size (the FCN step: six GEMMs of
    # 3.4e10 flop, each ~12 us slower when bracketed) times a rotating one of them
    eligible = sum(1 for _, m, n, k, _ in calls if 2.0 * m * n * k >= min_work)
    sample_every = eligible + 1 if args.workload == "fcn" and eligible > 1 else 1
    L.mtnn_profile_reset()
    L.mtnn_profile_enable_classes((1 << _lib.KCLASS_GEMM_TC) | (1 << _lib.KCLASS_GEMM_TC_F16S)
                                  | (1 << _lib.KCLASS_GEMM_FFMA))
    L.mtnn_profile_min_work(ctypes.c_double(min_work))
    L.mtnn_profile_sample_every(sample_every)
    events = []
    with clock_sampler(local_rank) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            one_step(events)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        wall = time.perf_counter() - w0
    L.mtnn_profile_enable(0)
    device_s = sum(s.elapsed_time(e) for s, e in events) * 1e-3
    t = torch.tensor([device_s], dtype=torch.float64,
                     device=dev if not share else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    device_s = float(t.item())
    step_s = device_s / args.steps
    value = total_flops / step_s / 1e12
    prof = {c: _lib.profile_read(c) for c in _lib.KCLASS_NAMES}
    prof_t = {c: _lib.profile_read_timed(c) for c in _lib.KCLASS_NAMES}
    launches = int(sum(v[1] for v in prof.values()))
    L.mtnn_profile_min_work(ctypes.c_double(0.0))
    L.mtnn_profile_sample_every(1)
    # per-class breakdown: one extra step with every launch timed
    L.mtnn_profile_reset()
    L.mtnn_profile_enable(1)
    one_step()
    torch.cuda.synchronize()
    L.mtnn_profile_enable(0)
    prof_all = {c: _lib.profile_read(c) for c in _lib.KCLASS_NAMES}
    L.mtnn_profile_reset()
    ncall = len(calls)
    verify = None if args.no_verify else verify_step(calls, run_call, out_view, a_views, b_views,
                                                      grad_bufs, torch)
    if world > 1 and verify is not None:
        t = torch.tensor([verify["worst_rel_frobenius"], float(verify["failed"])],
                         dtype=torch.float64, device=dev if not share else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        verify.update({"worst_rel_frobenius": float(t[0]), "failed": int(t[1]),
                       "ranks": f"max over {world} ranks"})
    per_call = [statistics.median(events[st * (len(events) // args.steps) + i][0].elapsed_time(
        events[st * (len(events) // args.steps) + i][1]) for st in range(args.steps)) * 1e-3
        for i in range(len(events) // args.steps)]
    if world > 1 and args.workload == "large":
        # drop the collective windows (broadcast, and the all-gather unless fused)
        per_call = per_call[1:] if peer_gather is not None else per_call[1:-1]
    if world > 1 and args.workload == "fcn":
        per_call = per_call[:-1]

    # e2e through the host-buffer API: every rank runs its own cases (the sweep
    # at N > 1: its LPT share), the job time is the slowest rank's
    e2e = None
    if not args.no_e2e and (world == 1 or args.workload == "sweep"):
        if world > 1:
            dist.barrier()
        e2e = run_e2e(args, calls, handle, prefix_p, L)
        if world > 1:
            red = torch.tensor([e2e["ms_per_step"], float(e2e["h2d_bytes_per_step"]),
                                float(e2e["d2h_bytes_per_step"])], dtype=torch.float64,
                               device=dev if not share else "cpu")
            mx = red.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(red, op=dist.ReduceOp.SUM)
            ms = float(mx[0].item())
            e2e.update({"value": total_flops / (ms * 1e-3) / 1e12, "ms_per_step": ms,
                        "h2d_bytes_per_step": int(red[1].item()),
                        "d2h_bytes_per_step": int(red[2].item()),
                        "ranks": f"{world} ranks, each its own cases; max over ranks"})

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---------------- roofline of the dominant kernel
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(peaks_path.read_text()) if peaks_path.exists() else {}
    bf16 = peaks.get("bf16_tflops", 1590.0)
    # roof = the burst bf16 figure: the sweep step is 10s-100s of ms of GEMMs
    # separated by flushes and spin kernels, and boxes that stay cool run it above
    # the 4 s back-to-back "sustained" cuBLAS figure (frac > 1 seen), so only the
    # burst figure bounds it; the sustained fraction is listed beside it
    bf16_sus = peaks.get("bf16_tflops_sustained", bf16)
    hbm = peaks.get("hbm_gbs", 6650.0)
    tc_class = max((_lib.KCLASS_GEMM_TC_F16S, _lib.KCLASS_GEMM_TC), key=lambda c: prof_t[c][0])
    tc_ms, tc_n, tc_work = prof_t[tc_class]
    tc_all_n, tc_all_work = prof[tc_class][1], prof[tc_class][2]
    f16s = tc_class == _lib.KCLASS_GEMM_TC_F16S
    roof = bf16 / 3.0 if f16s else bf16 / 6.0
    roof_sus = bf16_sus / 3.0 if f16s else bf16_sus / 6.0
    ncu_path = ROOT / "profiles" / "ncu_summary.json"
    ncu_traffic = json.loads(ncu_path.read_text()).get("gemm_tc3x_traffic", {}) if ncu_path.exists() else {}
    dominant = max(prof_all, key=lambda c: prof_all[c][0])
    achieved = tc_work / (tc_ms * 1e-3) / 1e12 if tc_ms else None
    roofline = {
        "kernel": _lib.KCLASS_NAMES[tc_class], "bound": "tensor",
        "achieved": achieved, "peak": roof, "unit": "TFLOP/s",
        "frac": achieved / roof if achieved else None,
        "traffic": ncu_traffic.get("traffic"),
        "traffic_launch": ncu_traffic.get("launch"),
        "traffic_algorithmic_bytes": ncu_traffic.get("algorithmic_bytes"),
        "traffic_wave_floor_bytes": ncu_traffic.get("wave_floor_bytes"),
        "peak_basis": (f"FP32-accurate roof = measured bf16 dense {bf16} TFLOP/s (MEASURED_PEAKS.json, "
                       f"burst) / 3 MMAs per product (fp16 = bf16 rate)" if f16s else
                       f"3xTF32 FP32-accurate roof = measured bf16 dense {bf16} TFLOP/s "
                       f"(MEASURED_PEAKS.json, burst) / 2 (tf32 rate) / 3 (MMAs per product)"),
        "peak_sustained": roof_sus, "frac_of_sustained": achieved / roof_sus if achieved else None,
        "launches": tc_n, "avg_launch_ms": tc_ms / tc_n if tc_n else None,
        "timed_launches_note": (f"event-timed launches of >= {min_work:.3g} flop"
                                + (f", every {sample_every}th of those (rotating)" if sample_every > 1 else "")
                                + f": {tc_n} of {tc_all_n} launches of the class, "
                                f"{tc_work / tc_all_work:.1%} of its flops"
                                if tc_all_work else None),
        "share_of_step": tc_ms / 1e3 / (device_s * 1.0) if device_s else None,
        "dominant_kernel_by_time": _lib.KCLASS_NAMES[dominant],
    }
    kernels_summary = {_lib.KCLASS_NAMES[c]: {"ms": v[0], "launches_per_step": v[1],
                                              "work_per_step": v[2]}
                       for c, v in prof_all.items() if v[1]}
    kernels_summary["source"] = "one extra step with every launch timed (after the K timed steps)"

    extra = {}
    if args.workload == "sweep" and world == 1:
        extra.update(sweep_oracle_pass(shapes, per_call, ab_ptrs, C, flush_src, stream, handle,
                                       prefix_p, disp, total_flops, roof, args.oracle_reps, L, _lib,
                                       torch))
    if args.workload in ("large", "fcn") and world > 1:
        extra["collective_ms_per_step"] = {
            k: statistics.mean(s.elapsed_time(e) for s, e in v) for k, v in comm.items() if v}
        # compute-only view (§8e): the step without its separate collective
        # windows (this rank's); with the fused gather the C stores stay inside
        # the GEMM window, so only the broadcast of B is removed
        comm_ms = sum(extra["collective_ms_per_step"].values())
        comp_ms = step_s * 1e3 - comm_ms
        if comp_ms > 0:
            extra["compute_only"] = {
                "value": total_flops / (comp_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                "ms_per_step": comp_ms,
                "excludes": sorted(extra["collective_ms_per_step"]),
            }
    if gather_mode is not None:
        extra["gather"] = gather_mode
    if args.workload == "fcn":
        extra["per_call_us"] = {f"{op} ({m},{n},{k})#{i}": round(t * 1e6, 1)
                                for i, ((op, m, n, k, _), t) in enumerate(zip(calls, per_call))}
    if world == 1 and args.workload == "sweep":
        # a short idle first: the pass measures single transposes, not the power
        # state the preceding back-to-back sweep passes leave behind
        time.sleep(1.5)
        extra["transpose"] = transpose_pass(B, C, flush_src, stream, hbm, L, _lib, torch)
    extra["selector_native_ns_incl_ctypes"] = selector_cost(L, handle, prefix_p)
    ns = ctypes.c_double()
    if L.mtnn_select_cost_ns(handle, prefix_p, 1000000, ctypes.byref(ns)) == 0:
        extra["selector_native_ns"] = ns.value  # the C++ decision alone

    cpu = None
    if not args.no_cpu and world == 1 and args.workload != "large":
        cpu = cpu_baseline(args, host_threads())

    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f32", "data": "synthetic uniform[-1,1) fp32 operands, resident in HBM",
        "config": workload_config(args, world, desc_par),
        "wall_ms_per_step": wall / args.steps * 1e3, "calls_per_step_rank0": ncall,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks.summary(), "kernels": kernels_summary, "verify": verify,
    }
    line.update(extra)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def verify_step(calls, run_call, out_view, a_views, b_views, grad_bufs, torch, samples=16):
    """One untimed step that checks its own outputs: after every call, a
    sampled samples x samples block of C against float64 on the device."""
    gen = np.random.default_rng(0)
    worst, failed = 0.0, 0
    for i, (op, m, n, k, _) in enumerate(calls):
        if m <= 0:
            continue
        run_call(i, grad_bufs.get(i))
        rows = torch.from_numpy(np.sort(gen.choice(m, min(m, samples), replace=False))).cuda()
        cols = torch.from_numpy(np.sort(gen.choice(n, min(n, samples), replace=False))).cuda()
        a = a_views[i].index_select(0, rows).double()
        b = b_views[i]
        bsel = b.index_select(1, cols).double().t() if op == "nn" else b.index_select(0, cols).double()
        want = a @ bsel.t()
        got = out_view(i).index_select(0, rows).index_select(1, cols).double()
        err = float(torch.linalg.norm(got - want) / torch.linalg.norm(want))
        worst = max(worst, err) if err == err else float("inf")
        failed += not err <= 1e-5
    torch.cuda.synchronize()
    return {"cases": len(calls), "failed": failed, "worst_rel_frobenius": worst, "gate": 1e-5,
            "method": f"after each call, a sampled {samples}x{samples} block of C vs float64 "
                      f"(A rows . B rows) on the device"}


def sweep_oracle_pass(shapes, per_case_timed, ab_ptrs, C, flush_src, stream, handle, prefix_p,
                      disp, total_flops, roof, reps, L, _lib, torch):
    """MTNN (the dispatcher), NT and TNN per case, interleaved in ONE pass under
    the same instrumentation (GEMM launches event-timed, like the timed steps),
    the candidate order rotated per repetition, median of `reps`, L2 flushed
    before every window (reference bench.py:129-146 time_callables_interleaved).
    MTNN vs the per-case best of both paths comes from this pass alone."""
    import ctypes

    from paper_1702_03192_b200 import ProblemShape

    names = ("mtnn", "nt", "tnn")
    ev = {w: [[] for _ in shapes] for w in names}
    choice = ctypes.c_int()
    L.mtnn_profile_enable_classes((1 << _lib.KCLASS_GEMM_TC) | (1 << _lib.KCLASS_GEMM_TC_F16S)
                                  | (1 << _lib.KCLASS_GEMM_FFMA))
    for rep in range(reps):
        order = names[rep % 3:] + names[: rep % 3]
        for i, (m, n, k) in enumerate(shapes):
            pa, pb = ab_ptrs[i]
            for which in order:
                flush_src.sum()
                torch.cuda._sleep(SLEEP_CYCLES)
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                s.record()
                if which == "mtnn":
                    rc = L.mtnn_dispatch_gemm(handle, prefix_p, pa, pb, C.data_ptr(), m, n, k, -1, 0,
                                              stream, ctypes.byref(choice))
                elif which == "nt":
                    rc = L.mtnn_gemm_nt(pa, pb, C.data_ptr(), m, n, k, 0, stream)
                else:
                    rc = L.mtnn_gemm_tnn(pa, pb, C.data_ptr(), m, n, k, 0, -1, stream)
                e.record()
                _lib.check(rc)
                ev[which][i].append((s, e))
        torch.cuda.synchronize()
    L.mtnn_profile_enable(0)
    L.mtnn_profile_reset()
    t = {w: [statistics.median(s.elapsed_time(e) for s, e in evs) * 1e-3 for evs in ev[w]]
         for w in names}
    best = [min(x, y) for x, y in zip(t["nt"], t["tnn"])]
    ratio = [b_ / m_ for b_, m_ in zip(best, t["mtnn"])]
    picked_tnn = [disp.select(ProblemShape(*sh)).choice.value == "tnn" for sh in shapes]
    faster_tnn = [y < x for x, y in zip(t["nt"], t["tnn"])]
    large = [i for i, (m, n, k) in enumerate(shapes) if min(m, n, k) >= 4096]
    large_tf = (sum(2.0 * shapes[i][0] * shapes[i][1] * shapes[i][2] for i in large)
                / sum(per_case_timed[i] for i in large) / 1e12) if large else None
    return {
        "mtnn_vs_best_of_both": {
            "mean_per_case_ratio": float(np.mean(ratio)),
            "min_per_case_ratio": float(np.min(ratio)),
            "mtnn_tflops": total_flops / sum(t["mtnn"]) / 1e12,
            "always_nt_tflops": total_flops / sum(t["nt"]) / 1e12,
            "always_tnn_tflops": total_flops / sum(t["tnn"]) / 1e12,
            "best_of_both_tflops": total_flops / sum(best) / 1e12,
            "aggregate_ratio": sum(best) / sum(t["mtnn"]),
            "method": f"one pass, MTNN/NT/TNN interleaved per case (order rotated), median of "
                      f"{reps}, same instrumentation for all three",
        },
        "selector": {"accuracy_vs_measured_faster_path": float(np.mean(
                         [p == f for p, f in zip(picked_tnn, faster_tnn)])),
                     "tnn_faster_cases": int(sum(faster_tnn)),
                     "tnn_picked_cases": int(sum(picked_tnn))},
        "large_shapes_tflops": large_tf,
        "large_shapes_frac_of_roof": large_tf / roof if large_tf else None,
    }


def transpose_pass(B, C, flush_src, stream, hbm, L, _lib, torch):
    """Transpose bandwidth (config 3): 8*rows*cols bytes per launch, median of 5."""
    tshapes = [(2 ** e, 2 ** e) for e in range(7, 15)] + [
        (1000, 1000), (3000, 5000), (16384, 128), (128, 16384), (4097, 1023), (12345, 6789),
        (8191, 8193)]
    tshapes = [(r, c) for r, c in tshapes if r * c <= min(B.numel(), C.numel())]
    out = {}
    for (r, c) in tshapes:
        ev = []
        for _ in range(5):
            flush_src.sum()
            torch.cuda._sleep(SLEEP_CYCLES)
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            _lib.check(L.mtnn_transpose(B.data_ptr(), C.data_ptr(), r, c, stream))
            e.record()
            ev.append((s, e))
        torch.cuda.synchronize()
        tt = statistics.median(s.elapsed_time(e) * 1e-3 for s, e in ev)
        out[f"{r}x{c}"] = 8.0 * r * c / tt / 1e9
    big = [out[k] for k in ("4096x4096", "8192x8192", "16384x16384") if k in out]
    med = statistics.median(big) if big else None
    return {"gbs_by_shape": {k: round(v, 1) for k, v in out.items()}, "gbs_large_median": med,
            "peak_hbm_gbs": hbm, "frac_of_measured_hbm": med / hbm if med else None,
            "frac_of_8tbs_spec": med / 8000.0 if med else None}


def selector_cost(L, handle, prefix_p):
    import ctypes

    raw, ch, rs = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
    n = 20000
    t0 = time.perf_counter()
    for _ in range(n):
        L.mtnn_select(handle, prefix_p, 1024, 1024, 1024, 1 << 40, ctypes.byref(raw),
                      ctypes.byref(ch), ctypes.byref(rs))
    return (time.perf_counter() - t0) / n * 1e9


def run_e2e(args, calls, handle, prefix_p, L):
    """The same step through the reference-facing C-ABI with HOST buffers:
    mtnn_dispatch_gemm_host for NT calls, mtnn_gemm_nn_host for NN calls, each
    copying its operands in from pinned memory and its result out."""
    import ctypes

    import torch

    from paper_1702_03192_b200 import _lib

    max_a = max([m * k for _, m, n, k, _ in calls] + [1])
    max_b = max([n * k for _, m, n, k, _ in calls] + [1])
    max_c = max([m * n for _, m, n, k, _ in calls] + [1])
    ha = torch.empty(max_a, dtype=torch.float32).pin_memory().uniform_(-1, 1)
    hb = torch.empty(max_b, dtype=torch.float32).pin_memory().uniform_(-1, 1)
    hc = torch.empty(max_c, dtype=torch.float32).pin_memory()
    ch = ctypes.c_int()
    h2d = sum(4 * (m * k + n * k) for _, m, n, k, _ in calls)
    d2h = sum(4 * m * n for _, m, n, k, _ in calls)
    steps = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 2)

    def step():
        for (op, m, n, k, _) in calls:
            if op in ("nt", "grad"):
                rc = L.mtnn_dispatch_gemm_host(handle, prefix_p, ha.data_ptr(), hb.data_ptr(),
                                               hc.data_ptr(), m, n, k, -1, 0, ctypes.byref(ch))
            else:
                rc = L.mtnn_gemm_nn_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, 0)
            _lib.check(rc)

    step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = max((time.perf_counter() - t0) / steps, 1e-9)
    flops = sum(2.0 * m * n * k for _, m, n, k, _ in calls)
    return {"value": flops / dt / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3, "steps": steps,
            "api": "mtnn_dispatch_gemm_host / mtnn_gemm_nn_host (include/mtnn_b200.h), pinned host "
                   "buffers, H2D/compute/D2H pipelined inside each call"}


if __name__ == "__main__":
    main()
