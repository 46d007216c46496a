"""Kernel backend selection (mirror of reference ``mtnn/_backend.py:17-41``).

The reference resolves ``MTNN_BACKEND`` once at import to ``numba`` or
``numpy``. This package has exactly one backend — the sm_100a CUDA library
``libmtnn_b200.so`` — so the accepted values are ``auto`` (default) and
``b200``; anything else raises ``ValueError`` naming the variable, as the
reference does. There is deliberately no CPU fallback: if the library is
missing, importing the package fails loudly.
"""

import os

_requested = os.environ.get("MTNN_BACKEND", "auto").strip().lower() or "auto"

if _requested not in ("auto", "b200"):
    raise ValueError(f"MTNN_BACKEND must be 'b200' or 'auto', got {_requested!r}")

BACKEND = "b200"


def active_backend() -> str:
    """Name of the kernel backend picked at import: always 'b200'."""
    return BACKEND
