"""MTNN B200 benchmark — BASELINE.json's metric on its sweep configuration.

Workload (configs[1]): the NT sweep m, n, k in {128, ..., 16384} (512 cases),
every case computed C = A B^T through the MTNN dispatcher (GBDT decision in
host C++, then the direct-NT or the TNN path on sm_100a). One "step" = one pass
over all cases. `value` = total flops / total device time (whole job), inputs
resident in HBM, L2 flushed (256 MiB write) before every case and excluded from
the timed windows. `e2e` = the same sweep through the reference-facing C-ABI
with pinned HOST buffers (H2D of A and B, D2H of C inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU, NCCL): every case is row-sharded — rank r
computes its m/N rows of C against the replicated B, with no collective in the
timed region (strong scaling: the total work is fixed). `--gather` adds the
NCCL all-gather of C. `--impl reference` times the reference's CPU
implementation of the path (the C restatement in oracle/, all host threads) on a
bounded sample of the same sweep.
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
def cpu_sample_run(shapes, threads, seed=0):
    """Reference CPU path (oracle port of the numba kernels) over `shapes`:
    NT (row-dot) and TNN (transpose + blocked NN) per case, all `threads`;
    returns (flops, seconds of the per-case best path, seconds NT, seconds TNN)."""
    import oracle

    flops = secs_best = secs_nt = secs_tnn = 0.0
    for (m, n, k) in shapes:
        a, b, _ = oracle.make_operands(m, n, k, seed)
        t0 = time.perf_counter()
        oracle.gemm_nt(a, b, threads=threads)
        t1 = time.perf_counter()
        oracle.gemm_tnn(a, b, threads=threads)
        t2 = time.perf_counter()
        flops += 2.0 * m * n * k
        secs_nt += t1 - t0
        secs_tnn += t2 - t1
        secs_best += min(t1 - t0, t2 - t1)
    return flops, secs_best, secs_nt, secs_tnn


def cpu_sample_shapes(max_seconds_hint: float):
    # the 2^7..2^11 sub-grid (125 cases, 1.25e11 flop per path) the survey timed
    # the reference on: ~10-30 s of CPU work; the full 2^7..2^14 grid would be
    # hours of CPU time.
    return grid(7, 11)


def host_threads() -> int:
    """All host cores this process may run on (torchrun sets OMP_NUM_THREADS=1,
    so the OpenMP default is not the machine's core count)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(threads: int):
    shapes = cpu_sample_shapes(20.0)
    cpu_sample_run(shapes[:8], threads)  # warm caches / thread pool
    flops, best, s_nt, s_tnn = cpu_sample_run(shapes, threads)
    return {
        "value": flops / best / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "port",
        "sample": (f"sweep sub-grid m,n,k in {{128..2048}} ({len(shapes)} cases), oracle/ C port of "
                   f"the reference numba kernels, best of NT/TNN per case (upper bound of the CPU "
                   f"MTNN), {threads} threads; always-NT {flops / s_nt / 1e12:.4f}, "
                   f"always-TNN {flops / s_tnn / 1e12:.4f} TFLOP/s"),
        "seconds": best,
    }


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path (oracle
    port), timed on the host cores; rank 0 only."""
    if rank != 0:
        return
    threads = host_threads()
    shapes = cpu_sample_shapes(20.0)
    for _ in range(args.warmup):
        cpu_sample_run(shapes[:16], threads)
    times, flops = [], 0.0
    for _ in range(args.steps):
        f, best, _, _ = cpu_sample_run(shapes, threads)
        times.append(best)
        flops = f
    value = flops * args.steps / sum(times) / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(times) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "nt_sweep (bounded CPU sample of configs[1])",
                   "cases": len(shapes), "sample": "m,n,k in {128..2048}"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                         "sample": f"sweep sub-grid m,n,k in {{128..2048}} ({len(shapes)} cases), "
                                   "best of NT/TNN per case, oracle/ C port of the reference kernels"},
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


def build_workload(args, rank, world):
    """Per-step call list for this rank: (op, m, n, k, flush_before).
    op: "nt" = MTNN-dispatched NT, "nn" = NN product, "grad" = an FCN weight-gradient
    NT (MTNN-dispatched into its own buffer; all-reduced across ranks when N > 1)."""
    if args.workload == "sweep":
        shapes = grid(args.exp_min, args.exp_max)
        owner = lpt_assign([2.0 * m * n * k for m, n, k in shapes], world)
        calls = [("nt", m, n, k, True) for (m, n, k), o in zip(shapes, owner) if o == rank]
        desc = (f"nt_sweep m,n,k in {{2^{args.exp_min}..2^{args.exp_max}}} ({len(shapes)} cases), "
                f"MTNN-selected (configs[1])")
        total = sum(2.0 * m * n * k for m, n, k in shapes)
        par = "single GPU" if world == 1 else f"cases LPT-sharded over {world} GPUs (no collective)"
        return calls, total, desc, "strong", par, shapes
    if args.workload == "fcn":
        hidden, batch, din0, dout_last = (4096,) * 3, 1024, 784, 10
        widths = [din0, *hidden, dout_last]
        layers = list(zip(widths[:-1], widths[1:]))
        calls = [("nt", batch, dout, din, i == 0) for i, (din, dout) in enumerate(layers)]
        for j, (din, dout) in enumerate(reversed(layers)):
            calls.append(("nn", batch, din, dout, j == 0))
            calls.append(("grad", dout, din, batch, False))  # weight gradient (an NT)
        total = sum(2.0 * m * n * k for _, m, n, k, _ in calls) * world
        desc = ("fcn_step 784-4096-4096-4096-10 batch 1024 (configs[3]): 4 forward NT + 4 backward "
                "NN + 4 backward NT, all NT through MTNN (the reference routes only forward NT)")
        par = ("single GPU" if world == 1 else
               f"data parallel x{world}: batch 1024 per GPU, weight gradients all-reduced (NCCL, "
               f"overlapped with the remaining backward GEMMs)")
        return calls, total, desc, ("weak" if world > 1 else "strong"), par, None
    # large (config 5): m = 65536 rows of A sharded, B replicated
    from paper_1702_03192_b200.sharding import row_range

    m, n, k = 65536, 8192, 8192
    lo, hi = row_range(m, rank, world)
    calls = [("nt", hi - lo, n, k, True)]
    desc = "large_nt m=65536 n=k=8192 (configs[4]), rows of A sharded, B replicated"
    par = ("single GPU" if world == 1 else
           f"row-sharded x{world}: NCCL broadcast of B, then the all-gather of C "
           + ("fused into the GEMM epilogue (peer stores over NVLink)" if args.gather == "fused"
              else "by ncclAllGather"))
    return calls, 2.0 * m * n * k, desc, "strong", par, None


# ----------------------------------------------------------------- GPU legs
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="sweep", choices=("sweep", "fcn", "large"))
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
    calls, total_flops, desc, scaling, par, shapes = build_workload(args, rank, world)

    # model: the B200-trained selector if present, else an empty model (always NT)
    if Path(args.model).exists():
        model = gbdt.load_model(args.model)
        model_name = Path(args.model).name
    else:
        model = gbdt.GbdtModel(trees=(), params=gbdt.GbdtParams(), n_features=8)
        model_name = "empty (always NT)"
    disp = Dispatcher(model, probe_platform())
    handle = disp._native.handle
    prefix_p = disp._prefix_p

    # resident synthetic operands; every call views prefixes of these buffers
    cap_a = max([m * k for _, m, n, k, _ in calls] + [1])
    cap_b = max([n * k for _, m, n, k, _ in calls] + [1])
    cap_c = max([m * n for _, m, n, k, _ in calls] + [1])
    if args.workload == "large":
        cap_c = 65536 * 8192  # gathered C
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    A = torch.rand(cap_a, device=dev, generator=g).mul_(2).sub_(1)
    B = torch.rand(cap_b, device=dev, generator=g).mul_(2).sub_(1)
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
            from paper_1702_03192_b200.sharding import PeerGather, row_range

            try:
                peer_gather = PeerGather(C[: 65536 * 8192].view(65536, 8192))
                large_row0 = row_range(65536, rank, world)[0]
            except Exception as exc:  # no IPC between these processes: NCCL fallback
                gather_mode = f"nccl (fused unavailable: {type(exc).__name__}: {exc})"[:200]
                peer_gather = None

    def run_call(op, m, n, k, out=None):
        if m <= 0:
            return
        if peer_gather is not None:
            peer_gather.gemm(A[: m * k].view(m, k), B[: n * k].view(n, k), large_row0, sync=False)
            return
        if op == "grad":
            rc = L.mtnn_dispatch_gemm(handle, prefix_p, A.data_ptr(), B.data_ptr(), out.data_ptr(),
                                      m, n, k, -1, 0, stream, ctypes.byref(choice))
        elif op == "nt":
            rc = L.mtnn_dispatch_gemm(handle, prefix_p, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                                      m, n, k, -1, 0, stream, ctypes.byref(choice))
        else:
            rc = L.mtnn_gemm_nn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, stream)
        if rc:
            _lib.check(rc)

    comm = {"bcast": [], "gather": [], "allreduce": []}

    from paper_1702_03192_b200.sharding import allreduce_weight_grad as allreduce_grad

    def one_step(events=None):
        if args.workload == "large" and world > 1:
            # B replicated from rank 0, timed as part of the sharded op
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
            dist.broadcast(B[: 8192 * 8192], src=0)
            ev[1].record()
            if events is not None:
                comm["bcast"].append(ev)
                events.append(ev)
        works = []
        for i, (op, m, n, k, fl) in enumerate(calls):
            if fl:
                flush_src.sum()
            # keep the GPU busy while the host enqueues the timed call, so the
            # event window holds device work only (no Python/ctypes gaps)
            torch.cuda._sleep(SLEEP_CYCLES)
            if events is not None:
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                s.record()
                run_call(op, m, n, k, grad_bufs.get(i))
                e.record()
                events.append((s, e))
            else:
                run_call(op, m, n, k, grad_bufs.get(i))
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
    L.mtnn_profile_reset()
    L.mtnn_profile_enable_classes((1 << _lib.KCLASS_GEMM_TC) | (1 << _lib.KCLASS_GEMM_TC_F16S)
                                  | (1 << _lib.KCLASS_GEMM_FFMA))
    L.mtnn_profile_min_work(ctypes.c_double(min_work))
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
    # per-class breakdown: one extra step with every launch timed
    L.mtnn_profile_reset()
    L.mtnn_profile_enable(1)
    one_step()
    torch.cuda.synchronize()
    L.mtnn_profile_enable(0)
    prof_all = {c: _lib.profile_read(c) for c in _lib.KCLASS_NAMES}
    L.mtnn_profile_reset()
    ncall = len(calls)
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
        "timed_launches_note": (f"event-timed launches of >= {min_work:.3g} flop: {tc_n} of {tc_all_n} "
                                f"launches of the class, {tc_work / tc_all_work:.1%} of its flops"
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
        extra.update(sweep_oracle_pass(shapes, per_call, A, B, C, flush_src, stream, disp,
                                       total_flops, roof, L, _lib, torch))
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
    if world == 1:
        # a short idle first: the pass measures single transposes, not the power
        # state the preceding back-to-back sweep passes leave behind
        time.sleep(1.5)
        extra["transpose"] = transpose_pass(B, C, flush_src, stream, hbm, L, _lib, torch)
    extra["selector_native_ns_incl_ctypes"] = selector_cost(L, handle, prefix_p)
    ns = ctypes.c_double()
    if L.mtnn_select_cost_ns(handle, prefix_p, 1000000, ctypes.byref(ns)) == 0:
        extra["selector_native_ns"] = ns.value  # the C++ decision alone

    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_baseline(host_threads())

    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f32", "data": "synthetic uniform[-1,1) fp32 operands, resident in HBM",
        "config": {"workload": desc, "calls_per_step": ncall, "model": model_name,
                   "l2": "flushed (256 MiB read) before every case/phase, outside the timed windows",
                   "parallelism": par,
                   "precision": ("FP32-accurate: 3 tensor-core MMAs per product on hi/lo operand "
                                 "halves (pow2-scaled FP16, or TF32) with FP32 promotion, or FP32 FFMA"),
                   "wall_ms_per_step": wall / args.steps * 1e3},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks.summary(), "kernels": kernels_summary,
    }
    line.update(extra)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def sweep_oracle_pass(shapes, per_case_mtnn, A, B, C, flush_src, stream, disp, total_flops, roof,
                      L, _lib, torch):
    """NT and TNN per case (median of 3, interleaved, same instrumentation as the
    timed steps): MTNN vs the per-case best of both paths, and selector accuracy."""
    from paper_1702_03192_b200 import ProblemShape

    nt_t, tnn_t = [[] for _ in shapes], [[] for _ in shapes]
    # the same instrumentation as the timed steps (GEMM launches timed only)
    L.mtnn_profile_enable_classes((1 << _lib.KCLASS_GEMM_TC) | (1 << _lib.KCLASS_GEMM_TC_F16S)
                                  | (1 << _lib.KCLASS_GEMM_FFMA))
    for _rep in range(3):
        for i, (m, n, k) in enumerate(shapes):
            for which in ("nt", "tnn"):
                flush_src.sum()
                torch.cuda._sleep(SLEEP_CYCLES)
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                s.record()
                if which == "nt":
                    _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, stream))
                else:
                    _lib.check(L.mtnn_gemm_tnn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, 0, -1,
                                               stream))
                e.record()
                (nt_t if which == "nt" else tnn_t)[i].append((s, e))
    torch.cuda.synchronize()
    L.mtnn_profile_enable(0)
    L.mtnn_profile_reset()
    nt_s = [statistics.median(s.elapsed_time(e) for s, e in ev) * 1e-3 for ev in nt_t]
    tnn_s = [statistics.median(s.elapsed_time(e) for s, e in ev) * 1e-3 for ev in tnn_t]
    best = [min(x, y) for x, y in zip(nt_s, tnn_s)]
    ratio = [b_ / m_ for b_, m_ in zip(best, per_case_mtnn)]
    picked_tnn = [disp.select(ProblemShape(*sh)).choice.value == "tnn" for sh in shapes]
    faster_tnn = [y < x for x, y in zip(nt_s, tnn_s)]
    large = [i for i, (m, n, k) in enumerate(shapes) if min(m, n, k) >= 4096]
    large_tf = (sum(2.0 * shapes[i][0] * shapes[i][1] * shapes[i][2] for i in large)
                / sum(per_case_mtnn[i] for i in large) / 1e12) if large else None
    return {
        "mtnn_vs_best_of_both": {"mean_per_case_ratio": float(np.mean(ratio)),
                                 "min_per_case_ratio": float(np.min(ratio)),
                                 "always_nt_tflops": total_flops / sum(nt_s) / 1e12,
                                 "always_tnn_tflops": total_flops / sum(tnn_s) / 1e12,
                                 "best_of_both_tflops": total_flops / sum(best) / 1e12},
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
