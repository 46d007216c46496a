"""The reference's 9-function kernel protocol, served by libmtnn_b200.so.

Drop-in for ``mtnn.kernels._numba_impl`` / ``_numpy_impl``
(/root/reference/pkg/src/mtnn/kernels/_numba_impl.py:103-222,
_numpy_impl.py:18-67): same names, same positional arguments, numpy in and a
fresh C-contiguous float32 numpy array out, inputs never written. Each call
goes through the C-ABI "_host" entry points (include/mtnn_b200.h), which copy
the operands to the B200, run the sm_100a kernels and copy the result back
before returning — the reference's synchronous semantics. ``block``/``tile``
are CPU cache-blocking hints with no meaning for the GPU kernels and are
accepted and ignored (as the reference's numpy backend does,
_numpy_impl.py:9-11). The ``*_parallel`` variants are the same GPU kernels.

Validation lives above the protocol (kernels/__init__.py), exactly as in the
reference; these functions assume C-contiguous 2-D float32 inputs.
"""

from __future__ import annotations

import numpy as np

from .. import _lib

F32 = np.float32
_VARIANT = _lib.VARIANT_AUTO


def _ptr(x: np.ndarray) -> int:
    return x.ctypes.data


def gemm_nn(a, b, block):
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=F32)
    _lib.check(_lib.lib.mtnn_gemm_nn_host(_ptr(a), _ptr(b), _ptr(c), m, n, k, _VARIANT))
    return c


def gemm_nn_parallel(a, b, block):
    return gemm_nn(a, b, block)


def gemm_nt(a, b):
    m, k = a.shape
    n = b.shape[0]
    c = np.empty((m, n), dtype=F32)
    _lib.check(_lib.lib.mtnn_gemm_nt_host(_ptr(a), _ptr(b), _ptr(c), m, n, k, _VARIANT))
    return c


def gemm_nt_parallel(a, b):
    return gemm_nt(a, b)


def transpose_oop(b, tile):
    n, k = b.shape
    out = np.empty((k, n), dtype=F32)
    _lib.check(_lib.lib.mtnn_transpose_host(_ptr(b), _ptr(out), n, k))
    return out


def gemm_tnn(a, b, block, tile):
    m, k = a.shape
    n = b.shape[0]
    c = np.empty((m, n), dtype=F32)
    _lib.check(_lib.lib.mtnn_gemm_tnn_host(_ptr(a), _ptr(b), _ptr(c), m, n, k, _VARIANT, -1))
    return c


def gemm_tnn_parallel(a, b, block, tile):
    return gemm_tnn(a, b, block, tile)


def _packed_args(feat, thresh, left, right, leaf):
    feat = np.ascontiguousarray(feat, dtype=np.int64)
    thresh = np.ascontiguousarray(thresh, dtype=np.float64)
    left = np.ascontiguousarray(left, dtype=np.int64)
    right = np.ascontiguousarray(right, dtype=np.int64)
    leaf = np.ascontiguousarray(leaf, dtype=np.float64)
    n_trees, width = feat.shape
    return (feat, thresh, left, right, leaf), (
        feat.ctypes.data_as(_lib._I64P), thresh.ctypes.data_as(_lib._DP),
        left.ctypes.data_as(_lib._I64P), right.ctypes.data_as(_lib._I64P),
        leaf.ctypes.data_as(_lib._DP), n_trees, width)


def walk_trees(feat, thresh, left, right, leaf, x, base_score, eta):
    keep, args = _packed_args(feat, thresh, left, right, leaf)
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(_lib.lib.mtnn_walk_trees(*args, x.ctypes.data_as(_lib._DP),
                                          float(base_score), float(eta)))


def walk_trees_mnk(feat, thresh, left, right, leaf, prefix, m, n, k, base_score, eta):
    keep, args = _packed_args(feat, thresh, left, right, leaf)
    prefix = np.ascontiguousarray(prefix, dtype=np.float64)
    return float(_lib.lib.mtnn_walk_trees_mnk(*args, prefix.ctypes.data_as(_lib._DP),
                                              float(m), float(n), float(k),
                                              float(base_score), float(eta)))
