"""Device-resident entry points over CUDA torch tensors.

torch is used only for buffers and the current stream; the compute is the
C-ABI of libmtnn_b200.so (device pointers + cudaStream_t). All functions are
asynchronous on the current torch stream, allocate their outputs with torch's
caching allocator unless ``out`` is given, and never write their inputs.
"""

from __future__ import annotations

import torch

from . import _lib

_L = _lib.lib


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _check(x, name):
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32
            and x.dim() == 2 and x.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous 2-D float32 CUDA tensor")


def _same_device(*xs):
    devs = {x.device for x in xs}
    if len(devs) != 1:
        raise ValueError(f"operands are on different devices: {sorted(map(str, devs))}")


def _inner(ka, kb, what):
    if ka != kb:
        raise ValueError(f"A and B must share k ({what}): {ka} vs {kb}")


def _out(out, m, n, like):
    if out is None:
        return torch.empty((m, n), dtype=torch.float32, device=like.device)
    _check(out, "out")
    if tuple(out.shape) != (m, n):
        raise ValueError(f"out has shape {tuple(out.shape)}, expected {(m, n)}")
    _same_device(out, like)
    return out


def gemm_nt(a, b, *, out=None, variant: int = _lib.VARIANT_AUTO):
    """C = A B^T, A (m x k), B (n x k)."""
    _check(a, "a"); _check(b, "b")
    _same_device(a, b)
    m, k = a.shape
    n = b.shape[0]
    _inner(k, b.shape[1], "NT: A is m x k, B is n x k")
    c = _out(out, m, n, a)
    with torch.cuda.device(a.device):
        _lib.check(_L.mtnn_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k,
                                   variant, _stream()))
    return c


def gemm_nn(a, bt, *, out=None, variant: int = _lib.VARIANT_AUTO):
    """C = A BT, A (m x k), BT (k x n)."""
    _check(a, "a"); _check(bt, "b")
    _same_device(a, bt)
    m, k = a.shape
    n = bt.shape[1]
    _inner(k, bt.shape[0], "NN: A is m x k, BT is k x n")
    c = _out(out, m, n, a)
    with torch.cuda.device(a.device):
        _lib.check(_L.mtnn_gemm_nn(a.data_ptr(), bt.data_ptr(), c.data_ptr(), m, n, k,
                                   variant, _stream()))
    return c


def gemm_tnn(a, b, *, out=None, variant: int = _lib.VARIANT_AUTO, mem_budget: int = -1):
    """C = A (B^T) through a stream-ordered B^T buffer: transpose + NN."""
    _check(a, "a"); _check(b, "b")
    _same_device(a, b)
    m, k = a.shape
    n = b.shape[0]
    _inner(k, b.shape[1], "TNN: A is m x k, B is n x k")
    c = _out(out, m, n, a)
    with torch.cuda.device(a.device):
        _lib.check(_L.mtnn_gemm_tnn(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k,
                                    variant, mem_budget, _stream()))
    return c


def transpose(b, *, out=None):
    """Out-of-place bit-exact transpose of a rows x cols tensor."""
    _check(b, "b")
    r, c = b.shape
    o = _out(out, c, r, b)
    with torch.cuda.device(b.device):
        _lib.check(_L.mtnn_transpose(b.data_ptr(), o.data_ptr(), r, c, _stream()))
    return o
