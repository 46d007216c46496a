"""Row-sharded NT across GPUs: C = A·Bᵀ with A and C split by rows.

Row i of C depends only on row i of A and all of B, so rank r of N owns rows
``row_range(m, r, N)`` of A and C; B is replicated (``ncclBroadcast`` from the
rank that holds it) and, when the caller wants the whole C everywhere, the
contiguous row blocks are reassembled with one ``ncclAllGather`` — the only two
exchange steps the path has. One process per GPU, ``torch.distributed`` with the
NCCL backend for the plumbing; the local product is the MTNN dispatcher (or a
fixed path) on this rank's GPU.

The reference has no distributed code (SPEC.md:213 lists multi-GPU sweeps as a
non-goal); this is the B200 build's scaling axis for config 5
(m = 65536, n = k = 8192 over 1/2/4/8 GPUs).
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def row_range(m: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) rows of an m-row matrix owned by `rank` (balanced, contiguous)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    return (m * rank) // world, (m * (rank + 1)) // world


def shard_rows(x: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    lo, hi = row_range(x.shape[0], rank, world)
    return x[lo:hi]


def _default_gemm(variant: str):
    from . import kernels

    return lambda a, b: kernels.gemm_nt(a, b, variant=variant)


def broadcast_b(b: torch.Tensor | None, shape, *, src: int = 0, group=None,
                device=None) -> torch.Tensor:
    """Replicate B (n x k) from `src` to every rank of `group`."""
    rank = dist.get_rank(group)
    if rank == src:
        if b is None:
            raise ValueError("source rank must provide B")
        out = b.contiguous()
    else:
        out = torch.empty(tuple(shape), dtype=torch.float32, device=device)
    dist.broadcast(out, src=dist.get_global_rank(group, src) if group is not None else src,
                   group=group)
    return out


def gather_rows(c_local: torch.Tensor, m: int, *, group=None) -> torch.Tensor:
    """All-gather contiguous row blocks into the full m x n C on every rank.

    Blocks differ by at most one row when N does not divide m; they are padded
    to the largest block for the collective and the padding is dropped.
    """
    world = dist.get_world_size(group)
    n = c_local.shape[1]
    sizes = [row_range(m, r, world) for r in range(world)]
    rows = max(hi - lo for lo, hi in sizes)
    if all(hi - lo == rows for lo, hi in sizes):
        out = torch.empty((m, n), dtype=c_local.dtype, device=c_local.device)
        dist.all_gather_into_tensor(out, c_local.contiguous(), group=group)
        return out
    padded = torch.zeros((rows, n), dtype=c_local.dtype, device=c_local.device)
    padded[: c_local.shape[0]] = c_local
    buf = torch.empty((world * rows, n), dtype=c_local.dtype, device=c_local.device)
    dist.all_gather_into_tensor(buf, padded, group=group)
    return torch.cat([buf[r * rows: r * rows + (hi - lo)] for r, (lo, hi) in enumerate(sizes)])


def sharded_gemm_nt(
    a_local: torch.Tensor,
    b: torch.Tensor | None,
    *,
    m: int,
    n: int,
    k: int,
    src: int = 0,
    gather: bool = True,
    group=None,
    gemm: Callable | None = None,
    variant: str = "auto",
) -> torch.Tensor:
    """Row-sharded C = A·Bᵀ.

    a_local: this rank's rows of A (``row_range(m, rank, N)``); b: B on rank
    `src` (ignored elsewhere; pass None), replicated by broadcast. Returns the
    full C (gather=True) or this rank's C rows. `gemm(a, b)` is the local NT
    product: by default the B200 MTNN NT path; any callable with the same
    contract (e.g. a Dispatcher's ``gemm``) works.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = row_range(m, rank, world)
    if tuple(a_local.shape) != (hi - lo, k):
        raise ValueError(f"rank {rank}: A block has shape {tuple(a_local.shape)}, "
                         f"expected {(hi - lo, k)}")
    b_rep = broadcast_b(b, (n, k), src=src, group=group, device=a_local.device)
    gemm = gemm or _default_gemm(variant)
    c_local = gemm(a_local, b_rep) if hi > lo else torch.empty((0, n), dtype=torch.float32,
                                                                 device=a_local.device)
    return gather_rows(c_local, m, group=group) if gather else c_local


# ------------------------------------------------------------------ FC layers
# Data-parallel FC training step (SURVEY §8e "FC batches"): each rank runs the
# layer GEMMs on its own batch rows — the forward NT (b_r, dout, din) is a
# row-sharded product with the weights replicated — and the weight-gradient NT
# (dout, din, b_r) contracts over the batch, so the per-rank partial gradients
# are summed by one all-reduce (the path's only exchange step besides B's
# replication).


def allreduce_weight_grad(grad: torch.Tensor, *, group=None, async_op: bool = True):
    """Sum a weight gradient over the ranks of `group`, in place.

    NCCL: asynchronous (returns the work handle; NCCL's stream waits for the
    GEMM that wrote `grad`, so later GEMMs overlap it — call ``wait()`` before
    using `grad`). Other backends (gloo test mode): synchronous through host
    memory, returns None.
    """
    if dist.get_backend(group) == "nccl":
        return dist.all_reduce(grad, group=group, async_op=async_op)
    t = grad.detach().cpu() if grad.is_cuda else grad
    dist.all_reduce(t, group=group)
    if t is not grad:
        grad.copy_(t)
    return None


def dp_weight_grad(dz_local: torch.Tensor, x_local: torch.Tensor, *, group=None,
                   gemm: Callable | None = None, variant: str = "auto") -> torch.Tensor:
    """dW = Σ_ranks dZ_rᵀ·X_r for one FC layer (dout x din).

    dz_local: this rank's (dout x b_r) output-gradient block (batch on columns,
    the reference's "nt-fixed" operand layout, fcn.py:191), x_local: its
    (din x b_r) input block. Local NT product (dout, din, b_r), then the
    all-reduce; returns the summed gradient on every rank.
    """
    gemm = gemm or _default_gemm(variant)
    g = gemm(dz_local.contiguous(), x_local.contiguous())
    work = allreduce_weight_grad(g, group=group)
    if work is not None:
        work.wait()
    return g


# ------------------------------------------------------- fused all-gather
class PeerGather:
    """Row-sharded NT with the all-gather fused into the GEMM.

    Every rank holds the full (m, n) C buffer `c`; at construction the ranks
    exchange CUDA IPC handles of their buffers (``all_gather_object`` over the
    process group — plumbing only) and map each other's. ``gemm(a_local, b,
    row0)`` then runs ``mtnn_gemm_nt_allgather``: the CTA-pair GEMM epilogue
    stores every C tile of this rank's row block into its own C and straight
    into each peer's C over NVLink, so the gather overlaps the MMAs instead of
    following them as an ``ncclAllGather``. Completion is a device-side barrier
    over IPC-mapped flag words (``mtnn_peer_barrier``) enqueued after the GEMM:
    once it passes on a rank's stream, that rank's C holds every rank's rows.
    """

    def __init__(self, c: torch.Tensor, *, group=None, timeout_s: float = 30.0):
        import ctypes

        from . import _lib

        if not (c.is_cuda and c.dtype == torch.float32 and c.is_contiguous() and c.dim() == 2):
            raise ValueError("c must be a contiguous 2-D float32 CUDA tensor")
        self.c, self.group, self.timeout_s = c, group, float(timeout_s)
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        if self.world > 8:
            raise ValueError("PeerGather maps at most 8 ranks (one NVSwitch node)")
        # per-rank flag words of the device-side barrier (slot i written by rank i)
        self.flags = torch.zeros(8, dtype=torch.int32, device=c.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=c.device)
        self.epoch = 0
        mine = []
        for t in (c, self.flags):
            handle = (ctypes.c_char * 64)()
            off = ctypes.c_int64()
            _lib.check(_lib.lib.mtnn_ipc_handle(t.data_ptr(), ctypes.addressof(handle),
                                                ctypes.byref(off)))
            mine.append((bytes(handle), off.value))
        infos = [None] * self.world
        dist.all_gather_object(infos, tuple(mine), group=group)
        self.peers, self.peer_flags = [], []
        for r, entries in enumerate(infos):
            if r == self.rank:
                continue
            for (h, o), dst in zip(entries, (self.peers, self.peer_flags)):
                buf = ctypes.create_string_buffer(h, 64)
                p = ctypes.c_void_p()
                _lib.check(_lib.lib.mtnn_ipc_open(ctypes.addressof(buf), o, ctypes.byref(p)))
                dst.append(p.value)
        self._peer_arr = (ctypes.c_void_p * max(1, len(self.peers)))(*self.peers)
        self._flag_arr = (ctypes.c_void_p * max(1, len(self.peer_flags)))(*self.peer_flags)

    def _barrier(self, stream):
        from . import _lib

        self.epoch += 1
        _lib.check(_lib.lib.mtnn_peer_barrier(
            self.flags.data_ptr(), self._flag_arr, len(self.peer_flags), self.rank, self.world,
            self.epoch & 0xFFFFFFFF, self.status.data_ptr(), self.timeout_s, stream))

    def check_status(self):
        """Raise if a device-side barrier timed out waiting for a peer."""
        bad = int(self.status.item())
        if bad:
            raise RuntimeError(f"PeerGather: rank {bad - 1} never reached the device barrier "
                               f"(timeout {self.timeout_s} s)")

    def gemm(self, a_local: torch.Tensor, b: torch.Tensor, row0: int, *, sync: bool = True):
        """Enqueue barrier -> fused GEMM + peer stores -> barrier on the current
        stream. The first barrier keeps this rank from storing into a peer's C
        while that peer's earlier work may still read it; the second makes C
        complete on this rank's stream (everything after it sees all ranks'
        tiles) without a host round trip. sync=True also waits on the host."""
        from . import _lib

        m, n = self.c.shape
        mloc, k = a_local.shape
        if tuple(b.shape) != (n, k) or row0 < 0 or row0 + mloc > m:
            raise ValueError(f"shapes: a_local {tuple(a_local.shape)}, b {tuple(b.shape)}, "
                             f"row0 {row0}, C {tuple(self.c.shape)}")
        if a_local.device != self.c.device or b.device != self.c.device:
            raise ValueError("a_local, b and c must be on the same device")
        # bound for the duration of the (asynchronous) launch: a temporary made
        # by .contiguous() must not return to the caching allocator before the
        # kernel has read it
        a_c, b_c = a_local.contiguous(), b.contiguous()
        stream = torch.cuda.current_stream(self.c.device)
        sp = stream.cuda_stream
        self._barrier(sp)
        _lib.check(_lib.lib.mtnn_gemm_nt_allgather(
            a_c.data_ptr(), b_c.data_ptr(), self.c.data_ptr(),
            self._peer_arr, len(self.peers), row0, mloc, n, k, sp))
        self._barrier(sp)
        for t in (a_c, b_c):
            if t is not a_local and t is not b:
                t.record_stream(stream)
        if sync:
            torch.cuda.synchronize(self.c.device)
            self.check_status()
        return self.c

    def close(self):
        from . import _lib

        torch.cuda.synchronize(self.c.device)
        dist.barrier(group=self.group)  # no peer still stores into our buffers
        for p in self.peers + self.peer_flags:
            _lib.check(_lib.lib.mtnn_ipc_close(p))
        self.peers, self.peer_flags = [], []
