"""ctypes binding of libmtnn_b200.so (the C-ABI in include/mtnn_b200.h).

The library is the only compute path: if it is missing this module raises on
import (there is no CPU fallback), and calls that need a GPU fail with the
library's own error message when none is present.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_size_t, c_void_p
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libmtnn_b200.so"

OK = 0
EINVAL = 22
ENOMEM = 12
ECUDA = 5
ENOTSUP = 95

VARIANT_AUTO = 0
VARIANT_TC3XTF32 = 1
VARIANT_FFMA = 2
VARIANT_TC3XF16S = 3
VARIANTS = {"auto": VARIANT_AUTO, "tc3xtf32": VARIANT_TC3XTF32, "ffma": VARIANT_FFMA,
            "tc3xf16s": VARIANT_TC3XF16S}

KCLASS_GEMM_TC = 0
KCLASS_GEMM_FFMA = 1
KCLASS_TRANSPOSE = 2
KCLASS_SPLIT = 3
KCLASS_REDUCE = 4
KCLASS_GEMM_TC_F16S = 5
KCLASS_FIXUP = 6
KCLASS_NAMES = {0: "gemm_tc3xtf32", 1: "gemm_ffma", 2: "transpose", 3: "operand_split",
                4: "splitk_reduce", 5: "gemm_tc3xf16s", 6: "residual_fixup"}

CHOICE_NT = 0
CHOICE_TNN = 1
REASON_PREDICTED = 0
REASON_MEMORY_FALLBACK = 1

_F = POINTER(ctypes.c_float)
_I64P = POINTER(c_int64)
_DP = POINTER(c_double)


class MtnnError(RuntimeError):
    """A CUDA/runtime failure reported by libmtnn_b200."""


# diagnostics-only entry points a library selected by MTNN_B200_LIB may lack
_DIAGNOSTIC = {"mtnn_profile_trace", "mtnn_gate"}


def _load():
    path = os.environ.get("MTNN_B200_LIB", str(LIB_PATH))
    if not Path(path).exists():
        raise ImportError(
            f"libmtnn_b200.so not found at {path}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the B200 backend)"
        )
    lib = ctypes.CDLL(path)
    sig = {
        "mtnn_abi_version": (c_int, []),
        "mtnn_last_error": (c_char_p, []),
        "mtnn_device_available": (c_int, []),
        "mtnn_device_free_bytes": (c_int, [_I64P]),
        "mtnn_device_features": (c_int, [_DP]),
        "mtnn_profile_enable": (c_int, [c_int]),
        "mtnn_profile_enable_classes": (c_int, [ctypes.c_uint]),
        "mtnn_profile_reset": (c_int, []),
        "mtnn_profile_read": (c_int, [c_int, _DP, _I64P, _DP]),
        "mtnn_profile_read_timed": (c_int, [c_int, _DP, _I64P, _DP]),
        "mtnn_profile_min_work": (c_int, [ctypes.c_double]),
        "mtnn_profile_sample_every": (c_int, [c_int]),
        "mtnn_profile_trace": (c_int, [ctypes.c_void_p, ctypes.c_int64]),
        "mtnn_gate": (c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
        "mtnn_config_set": (c_int, [c_char_p, c_int64]),
        "mtnn_fill_uniform_pcg64": (c_int, [c_void_p, c_int64, POINTER(ctypes.c_uint64), c_int64,
                                            c_double, c_double, c_void_p]),
        "mtnn_config_get": (c_int, [c_char_p, _I64P]),
        "mtnn_gemm_nt_allgather": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(c_void_p), c_int,
                                           c_int64, c_int64, c_int64, c_int64, c_void_p]),
        "mtnn_ipc_handle": (c_int, [c_void_p, c_void_p, _I64P]),
        "mtnn_ipc_open": (c_int, [c_void_p, c_int64, POINTER(c_void_p)]),
        "mtnn_ipc_close": (c_int, [c_void_p]),
        "mtnn_peer_barrier": (c_int, [c_void_p, POINTER(c_void_p), c_int, c_int, c_int,
                                      ctypes.c_uint32, c_void_p, c_double, c_void_p]),
        "mtnn_gemm_nt": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p]),
        "mtnn_gemm_nn": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p]),
        "mtnn_transpose": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p]),
        "mtnn_gemm_tnn": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_int64, c_void_p]),
        "mtnn_gemm_nt_host": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int]),
        "mtnn_gemm_nn_host": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int]),
        "mtnn_transpose_host": (c_int, [c_void_p, c_void_p, c_int64, c_int64]),
        "mtnn_gemm_tnn_host": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_int64]),
        "mtnn_walk_trees": (c_double, [_I64P, _DP, _I64P, _I64P, _DP, c_int64, c_int64, _DP, c_double, c_double]),
        "mtnn_walk_trees_mnk": (c_double, [_I64P, _DP, _I64P, _I64P, _DP, c_int64, c_int64, _DP,
                                           c_double, c_double, c_double, c_double, c_double]),
        "mtnn_model_load_json": (c_int, [c_char_p, c_size_t, POINTER(c_void_p)]),
        "mtnn_model_from_packed": (c_int, [_I64P, _DP, _I64P, _I64P, _DP, c_int64, c_int64,
                                           c_double, c_double, c_int64, POINTER(c_void_p)]),
        "mtnn_model_free": (None, [c_void_p]),
        "mtnn_model_n_features": (c_int64, [c_void_p]),
        "mtnn_model_n_trees": (c_int64, [c_void_p]),
        "mtnn_model_raw": (c_int, [c_void_p, _DP, c_int64, _DP]),
        "mtnn_select": (c_int, [c_void_p, _DP, c_int64, c_int64, c_int64, c_int64, _DP,
                                POINTER(c_int), POINTER(c_int)]),
        "mtnn_select_cost_ns": (c_int, [c_void_p, _DP, c_int64, _DP]),
        "mtnn_dispatch_gemm": (c_int, [c_void_p, _DP, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                       c_int64, c_int64, c_int, c_void_p, POINTER(c_int)]),
        "mtnn_dispatch_gemm_host": (c_int, [c_void_p, _DP, c_void_p, c_void_p, c_void_p, c_int64,
                                            c_int64, c_int64, c_int64, c_int, POINTER(c_int)]),
    }
    for name, (res, args) in sig.items():
        if name in _DIAGNOSTIC and not hasattr(lib, name):
            continue  # (an older library under MTNN_B200_LIB for A/B runs)
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.mtnn_abi_version() != 1:
        raise ImportError(f"libmtnn_b200 ABI version {lib.mtnn_abi_version()} != 1")
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.mtnn_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception taxonomy."""
    if rc == OK:
        return
    msg = last_error()
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise MtnnError(msg or f"libmtnn_b200 error {rc}")


def profile_read(kclass: int):
    """(total_ms, launches, work) accumulated for one kernel class."""
    ms, n, w = ctypes.c_double(), c_int64(), ctypes.c_double()
    check(lib.mtnn_profile_read(kclass, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(w)))
    return ms.value, n.value, w.value


def profile_read_timed(kclass: int):
    """(total_ms, launches, work) of the timed launches of one kernel class (those
    with work >= the mtnn_profile_min_work threshold)."""
    ms, n, w = ctypes.c_double(), c_int64(), ctypes.c_double()
    check(lib.mtnn_profile_read_timed(kclass, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(w)))
    return ms.value, n.value, w.value


def config_set(key: str, value: int) -> None:
    check(lib.mtnn_config_set(key.encode(), int(value)))


def config_get(key: str) -> int:
    v = c_int64()
    check(lib.mtnn_config_get(key.encode(), ctypes.byref(v)))
    return v.value


def exported_symbols() -> list[str]:
    return [n for n in dir(lib) if n.startswith("mtnn_")]
