"""Apply INTEGRATION.md §1-3 to a COPY of the installed reference package.

Test infrastructure: copies baseline/_ref/mtnn (the unmodified reference,
installed by tools/install_reference.sh) into a scratch directory and makes
exactly the maintainer edits INTEGRATION.md documents:

  §1 _backend.py accepts MTNN_BACKEND=b200 and sets BACKEND = "b200";
  §2 kernels/__init__.py and selector.py bind ``_impl`` to ``_b200_impl``;
  §3 kernels/_b200_impl.py is the ctypes stub — here it re-exports this
     repository's paper_1702_03192_b200.kernels._b200_impl (the same module
     INTEGRATION.md §3 lists).

Every edit anchors on the reference's own source text and fails loudly if it
is not found, so a changed reference cannot be silently half-bound.
"""

from __future__ import annotations

import shutil
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"


def _edit(path: Path, old: str, new: str) -> None:
    text = path.read_text()
    if old not in text:
        raise RuntimeError(f"{path}: anchor not found: {old[:60]!r}")
    path.write_text(text.replace(old, new, 1))


def bind(dst: Path) -> Path:
    """dst/mtnn = reference package bound to the B200 backend; returns dst."""
    src = REF / "mtnn"
    if not src.is_dir():
        raise FileNotFoundError(f"{src} missing: run tools/install_reference.sh")
    pkg = dst / "mtnn"
    shutil.copytree(src, pkg, ignore=shutil.ignore_patterns("__pycache__"))
    _edit(pkg / "_backend.py",
          'if _requested not in ("auto", "numba", "numpy"):',
          'if _requested not in ("auto", "numba", "numpy", "b200"):')
    _edit(pkg / "_backend.py",
          'BACKEND = "numba" if HAS_NUMBA else "numpy"',
          'BACKEND = "b200" if _requested == "b200" else ("numba" if HAS_NUMBA else "numpy")')
    _edit(pkg / "kernels" / "__init__.py",
          'if BACKEND == "numba":\n    from . import _numba_impl as _impl',
          'if BACKEND == "b200":\n    from . import _b200_impl as _impl\n'
          'elif BACKEND == "numba":\n    from . import _numba_impl as _impl')
    _edit(pkg / "selector.py",
          'if kernels.BACKEND == "numba":\n    from .kernels import _numba_impl as _impl',
          'if kernels.BACKEND == "b200":\n    from .kernels import _b200_impl as _impl\n'
          'elif kernels.BACKEND == "numba":\n    from .kernels import _numba_impl as _impl')
    (pkg / "kernels" / "_b200_impl.py").write_text(
        '"""INTEGRATION.md §3: the B200 ctypes stub (this repository\'s module)."""\n'
        "from paper_1702_03192_b200.kernels._b200_impl import *  # noqa: F401,F403\n"
        "from paper_1702_03192_b200.kernels._b200_impl import (  # noqa: F401\n"
        "    gemm_nn, gemm_nn_parallel, gemm_nt, gemm_nt_parallel, gemm_tnn, gemm_tnn_parallel,\n"
        "    transpose_oop, walk_trees, walk_trees_mnk)\n")
    return dst
