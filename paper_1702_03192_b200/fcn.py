"""Fully-connected-network GEMM workload on the B200.

GPU restatement of the reference's FCN emulation
(/root/reference/pkg/src/mtnn/fcn.py): one training iteration is its GEMM
call sequence on seeded operands — per layer with ``din`` inputs, ``dout``
outputs and mini-batch ``b``:

- forward: NT ``(b, dout, din)``, activations x weightsᵀ — the call the
  dispatcher intercepts (fcn.py:166-178);
- backward: NN ``(b, din, dout)`` input gradient (fcn.py:183) and the NT
  weight-gradient stand-in ``(dout, din, b)`` (fcn.py:191).

Operands are generated with the reference's RNG order (``default_rng(seed)``;
x, w, dz, ga, gb per layer, fcn.py:122-147) and kept resident on the GPU; each
GEMM is timed with CUDA events on the current stream, with an L2 flush (a
256 MiB read) before each phase in place of the reference's cache-normalising
``_touch``. The reference routes only the forward NT through the dispatcher
and runs the weight-gradient NT as a fixed kernel ("nt-fixed");
``backward_nt="dispatch"`` routes it through MTNN as well — BASELINE config 4
("all NT ops routed through MTNN") uses that, and says so.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import kernels
from .selector import Dispatcher

__all__ = [
    "GemmCall",
    "FcnResult",
    "FcnInfeasibleError",
    "PRESETS",
    "DEFAULT_BATCHES",
    "preset_widths",
    "scaled_widths",
    "fcn_scenario",
    "compare_dispatchers",
    "iteration_flops",
]

# preset -> (input_dim, output_dim, {hidden_layer_count: widths}) (fcn.py:44-55)
PRESETS = {
    "mnist-like": (784, 10, {
        2: (2048, 1024),
        3: (2048, 2048, 1024),
        4: (2048, 2048, 2048, 1024),
    }),
    "synthetic-like": (26752, 26752, {
        2: (4096, 4096),
        3: (4096, 4096, 4096),
        4: (4096, 4096, 4096, 4096),
    }),
}
DEFAULT_BATCHES = {"mnist-like": (8, 16), "synthetic-like": (32, 64, 128)}


class FcnInfeasibleError(ValueError):
    """A layer's operands do not fit the device-memory budget."""


@dataclass(frozen=True)
class GemmCall:
    phase: str  # "forward" or "backward"
    op: str     # "nt" (dispatchable), "nn" or "nt-fixed"
    m: int
    n: int
    k: int
    seconds: float


@dataclass(frozen=True)
class FcnResult:
    forward_seconds: float
    backward_seconds: float
    calls: tuple

    @property
    def total_seconds(self) -> float:
        return self.forward_seconds + self.backward_seconds


def preset_widths(preset: str, hidden_layers: int):
    if preset not in PRESETS:
        raise ValueError(f"unknown preset {preset!r}; choose from {sorted(PRESETS)}")
    input_dim, output_dim, by_depth = PRESETS[preset]
    if hidden_layers not in by_depth:
        raise ValueError(f"preset {preset!r} supports {sorted(by_depth)} hidden layers, "
                         f"got {hidden_layers}")
    return input_dim, output_dim, by_depth[hidden_layers]


def scaled_widths(widths: Sequence[int], divisor: int) -> tuple:
    if divisor < 1:
        raise ValueError(f"scale divisor must be >= 1, got {divisor}")
    return tuple(max(1, w // divisor) for w in widths)


def _widths(hidden, input_dim, output_dim):
    widths = [int(input_dim)] + [int(w) for w in hidden] + [int(output_dim)]
    if any(w < 1 for w in widths):
        raise ValueError(f"layer widths must be positive, got {widths}")
    return widths


def iteration_flops(hidden, batch, input_dim, output_dim) -> int:
    """2*m*n*k summed over the 3 GEMMs per layer of one iteration."""
    widths = _widths(hidden, input_dim, output_dim)
    return sum(3 * 2 * batch * din * dout for din, dout in zip(widths[:-1], widths[1:]))


def _device_budget(mem_fraction: float) -> float:
    from .selector import _free_memory_bytes

    return _free_memory_bytes() * mem_fraction


def _build_layers(hidden, batch, input_dim, output_dim, seed, mem_fraction, device):
    import torch

    if batch < 1:
        raise ValueError(f"batch must be >= 1, got {batch}")
    widths = _widths(hidden, input_dim, output_dim)
    budget = _device_budget(mem_fraction)
    rng = np.random.default_rng(seed)
    layers = []
    for index, (din, dout) in enumerate(zip(widths[:-1], widths[1:])):
        need = 4 * (batch * din + 2 * dout * din + 2 * batch * dout + dout * din)
        if need > budget:
            raise FcnInfeasibleError(
                f"layer {index} ({din} -> {dout}, batch {batch}) needs {need / 2**20:.0f} MiB, "
                f"budget is {budget / 2**20:.0f} MiB; try a larger scale divisor")
        host = {
            "x": rng.uniform(-1, 1, (batch, din)).astype(np.float32),
            "w": rng.uniform(-1, 1, (dout, din)).astype(np.float32),
            "dz": rng.uniform(-1, 1, (batch, dout)).astype(np.float32),
            "ga": rng.uniform(-1, 1, (dout, batch)).astype(np.float32),
            "gb": rng.uniform(-1, 1, (din, batch)).astype(np.float32),
        }
        layer = {"din": din, "dout": dout}
        layer.update({k: torch.from_numpy(v).to(device) for k, v in host.items()})
        layers.append(layer)
    return layers


def _check_dispatch(dispatch):
    if isinstance(dispatch, str) and dispatch not in ("nt", "tnn"):
        raise ValueError(f"dispatch must be 'nt', 'tnn' or a Dispatcher, got {dispatch!r}")


def _nt_call(dispatch, a, b):
    if isinstance(dispatch, Dispatcher):
        return dispatch.gemm(a, b)
    if dispatch == "nt":
        return kernels.gemm_nt(a, b)
    return kernels.gemm_tnn(a, b)


class _Timer:
    """CUDA-event windows on the current stream, resolved after one sync."""

    def __init__(self):
        import torch

        self.torch = torch
        self.windows = []

    def run(self, label, fn):
        ev0 = self.torch.cuda.Event(enable_timing=True)
        ev1 = self.torch.cuda.Event(enable_timing=True)
        ev0.record()
        out = fn()
        ev1.record()
        self.windows.append((label, ev0, ev1))
        return out

    def resolve(self):
        self.torch.cuda.synchronize()
        return [(label, a.elapsed_time(b) * 1e-3) for label, a, b in self.windows]


def _flush(buf):
    if buf is not None:
        buf.sum()


def _run_iteration(layers, batch, dispatch, backward_nt, flush_buf, calls=None):
    timer = _Timer()
    _flush(flush_buf)
    for layer in layers:
        timer.run(("forward", "nt", batch, layer["dout"], layer["din"]),
                  lambda l=layer: _nt_call(dispatch, l["x"], l["w"]))
    _flush(flush_buf)
    for layer in reversed(layers):
        timer.run(("backward", "nn", batch, layer["din"], layer["dout"]),
                  lambda l=layer: kernels.gemm_nn(l["dz"], l["w"]))
        if backward_nt == "dispatch":
            timer.run(("backward", "nt", layer["dout"], layer["din"], batch),
                      lambda l=layer: _nt_call(dispatch, l["ga"], l["gb"]))
        else:
            timer.run(("backward", "nt-fixed", layer["dout"], layer["din"], batch),
                      lambda l=layer: kernels.gemm_nt(l["ga"], l["gb"]))
    fwd = bwd = 0.0
    for (phase, op, m, n, k), secs in timer.resolve():
        if phase == "forward":
            fwd += secs
        else:
            bwd += secs
        if calls is not None:
            calls.append(GemmCall(phase, op, m, n, k, secs))
    return fwd, bwd


def _flush_buffer(device):
    import torch

    return torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=device)


def fcn_scenario(
    hidden: Sequence[int],
    batch: int,
    input_dim: int,
    output_dim: int,
    dispatch,
    *,
    iters: int = 1,
    warmup: int = 1,
    seed: int = 0,
    block: int = kernels.DEFAULT_BLOCK,
    tile: int = kernels.DEFAULT_TILE,
    threads: int = 1,
    mem_fraction: float = 0.8,
    backward_nt: str = "fixed",
    device: str = "cuda",
) -> FcnResult:
    """Run the GEMM sequence of one training iteration on the GPU and time it.

    ``dispatch`` is "nt", "tnn" or a Dispatcher; times are averaged over
    ``iters`` iterations after ``warmup`` discarded ones; per-call seconds in
    the log come from the last timed iteration (reference fcn.py:208-247).
    """
    _check_dispatch(dispatch)
    if iters < 1:
        raise ValueError(f"iters must be >= 1, got {iters}")
    if backward_nt not in ("fixed", "dispatch"):
        raise ValueError(f"backward_nt must be 'fixed' or 'dispatch', got {backward_nt!r}")
    kernels._resolve_threads(threads)
    layers = _build_layers(hidden, batch, input_dim, output_dim, seed, mem_fraction, device)
    flush_buf = _flush_buffer(device)
    for _ in range(warmup):
        _run_iteration(layers, batch, dispatch, backward_nt, flush_buf)
    fwd_total = bwd_total = 0.0
    calls = []
    for _ in range(iters):
        calls = []
        fwd, bwd = _run_iteration(layers, batch, dispatch, backward_nt, flush_buf, calls)
        fwd_total += fwd
        bwd_total += bwd
    return FcnResult(forward_seconds=fwd_total / iters, backward_seconds=bwd_total / iters,
                     calls=tuple(calls))


def compare_dispatchers(
    dispatchers: dict,
    hidden: Sequence[int],
    batches: Sequence[int],
    input_dim: int,
    output_dim: int,
    *,
    iters: int = 3,
    warmup: int = 1,
    seed: int = 0,
    block: int = kernels.DEFAULT_BLOCK,
    tile: int = kernels.DEFAULT_TILE,
    threads: int = 1,
    mem_fraction: float = 0.8,
    backward_nt: str = "fixed",
    device: str = "cuda",
) -> dict:
    """{name: (forward, backward) seconds}, averaged over batch sizes, with
    interleaved rotated rounds and best-of-rounds (reference fcn.py:250-299)."""
    for dispatch in dispatchers.values():
        _check_dispatch(dispatch)
    if iters < 1:
        raise ValueError(f"iters must be >= 1, got {iters}")
    sums = {name: [0.0, 0.0] for name in dispatchers}
    flush_buf = _flush_buffer(device)
    for batch in batches:
        layers = _build_layers(hidden, batch, input_dim, output_dim, seed, mem_fraction, device)
        rounds = {name: ([], []) for name in dispatchers}
        for _ in range(warmup):
            for dispatch in dispatchers.values():
                _run_iteration(layers, batch, dispatch, backward_nt, flush_buf)
        order = list(dispatchers)
        for r in range(iters):
            for name in order[r % len(order):] + order[: r % len(order)]:
                fwd, bwd = _run_iteration(layers, batch, dispatchers[name], backward_nt, flush_buf)
                rounds[name][0].append(fwd)
                rounds[name][1].append(bwd)
        for name in dispatchers:
            sums[name][0] += min(rounds[name][0])
            sums[name][1] += min(rounds[name][1])
    scale = 1.0 / len(list(batches))
    return {name: (f * scale, b * scale) for name, (f, b) in sums.items()}
