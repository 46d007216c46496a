"""Platform features used as selector inputs (mirror of reference platform.py).

The reference describes the host with five numbers (platform.py:22-44):
gm (memory GB), sm (compute units), cc (clock MHz), mbw (memory bus width,
bits) and l2c (L2 KB), detected once with override > detect > default+warning
(:113-139). On B200 the same five slots describe the GPU the kernels run on,
read from ``cudaDeviceGetAttribute`` through the C-ABI
(``mtnn_device_features``): HBM GiB, SM count (148), max SM clock (MHz),
memory bus width (bits) and L2 size (KB). The paper's features are GPU
properties too (Table III), so this restores the original
meaning.
"""

from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass
from typing import Mapping

from . import _lib

log = logging.getLogger(__name__)

DEFAULTS = {"gm": 8.0, "sm": 4.0, "cc": 2000.0, "mbw": 64.0, "l2c": 1024.0}
FEATURE_NAMES = ("gm", "sm", "cc", "mbw", "l2c")


@dataclass(frozen=True)
class PlatformFeatures:
    """The five platform features, all strictly positive."""

    gm: float
    sm: float
    cc: float
    mbw: float
    l2c: float

    def __post_init__(self):
        for name in FEATURE_NAMES:
            value = getattr(self, name)
            if not value > 0:
                raise ValueError(f"platform feature {name} must be > 0, got {value}")

    def as_tuple(self) -> tuple:
        return (self.gm, self.sm, self.cc, self.mbw, self.l2c)


def detect_device_features() -> dict | None:
    """The current CUDA device's five features, or None without a usable GPU."""
    out = (ctypes.c_double * 5)()
    if _lib.lib.mtnn_device_features(out) != _lib.OK:
        return None
    return dict(zip(FEATURE_NAMES, (float(v) for v in out)))


def probe_platform(overrides: Mapping[str, float] | None = None) -> PlatformFeatures:
    """Device features with ``overrides`` applied: override, then detect, then
    the documented default (logged as a warning)."""
    overrides = dict(overrides or {})
    unknown = set(overrides) - set(FEATURE_NAMES)
    if unknown:
        raise ValueError(f"unknown platform override(s): {sorted(unknown)}")
    detected = None
    if len(overrides) < len(FEATURE_NAMES):
        detected = detect_device_features()
        if detected is None:
            log.warning("no sm_100 device detected (%s)", _lib.last_error())
    values = {}
    for name in FEATURE_NAMES:
        if name in overrides:
            values[name] = float(overrides[name])
        elif detected is not None and detected[name] > 0:
            values[name] = detected[name]
        else:
            log.warning("could not detect %s; using default %s", name, DEFAULTS[name])
            values[name] = DEFAULTS[name]
    return PlatformFeatures(**values)
