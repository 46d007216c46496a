"""Validation contract of the kernel API (mirrors reference
tests/test_kernels.py:53-65, 98-100, 155-161, 188-245): everything here fails
before any device work, so it runs without a GPU."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_1702_03192_b200 import kernels
from paper_1702_03192_b200.kernels import (ProblemShape, as_matrix, gemm_nn, gemm_nt, gemm_tnn,
                                           transpose_oop)


def rm(rng, r, c):
    return rng.uniform(-1, 1, (r, c)).astype(np.float32)


def test_dim_mismatch_names_dimensions(rng):
    with pytest.raises(ValueError, match="2x3.*4x5"):
        gemm_nn(rm(rng, 2, 3), rm(rng, 4, 5))


def test_rejects_wrong_dtype(rng):
    with pytest.raises(TypeError, match="float32"):
        gemm_nn(rng.uniform(size=(3, 3)), rm(rng, 3, 3))
    with pytest.raises(TypeError, match="float32"):
        gemm_nt(rng.uniform(size=(3, 3)), rm(rng, 3, 3))


def test_rejects_noncontiguous(rng):
    with pytest.raises(ValueError, match="contiguous"):
        gemm_nn(rm(rng, 6, 6)[:, ::2], rm(rng, 3, 3))


def test_width_mismatch(rng):
    with pytest.raises(ValueError, match="share k"):
        gemm_nt(rm(rng, 2, 3), rm(rng, 2, 4))
    with pytest.raises(ValueError, match="share k"):
        gemm_tnn(rm(rng, 2, 3), rm(rng, 2, 4))


def test_mem_budget_raises_before_allocation(rng):
    with pytest.raises(MemoryError, match="budget"):
        gemm_tnn(rm(rng, 8, 8), rm(rng, 8, 8), mem_budget=16)


def test_bad_hints_rejected(rng):
    with pytest.raises(ValueError, match="block"):
        gemm_nn(rm(rng, 3, 3), rm(rng, 3, 3), block=2)
    with pytest.raises(ValueError, match="tile"):
        transpose_oop(rm(rng, 3, 3), tile=0)
    with pytest.raises(ValueError, match="threads"):
        gemm_nt(rm(rng, 3, 3), rm(rng, 3, 3), threads=0)
    with pytest.raises(ValueError, match="variant"):
        gemm_nt(rm(rng, 3, 3), rm(rng, 3, 3), variant="wmma")


def test_problem_shape():
    assert ProblemShape(2, 3, 4).flops == 48
    ProblemShape(1, 1, 1).validate()
    with pytest.raises(ValueError):
        ProblemShape(0, 1, 1).validate()


def test_as_matrix(rng):
    m = as_matrix([[1, 2], [3, 4]])
    assert m.dtype == np.float32 and m.flags.c_contiguous
    m = as_matrix(rng.uniform(size=(6, 6))[:, ::2])
    assert m.flags.c_contiguous and m.shape == (6, 3)
    with pytest.raises(ValueError, match="2-D"):
        as_matrix([1.0, 2.0])


def _run(env_value):
    env = dict(os.environ, MTNN_BACKEND=env_value, PYTHONPATH=str(ROOT))
    return subprocess.run([sys.executable, "-c",
                           "import paper_1702_03192_b200 as m; print(m.active_backend())"],
                          capture_output=True, text=True, env=env, cwd=str(ROOT))


def test_env_flag_selects_backend():
    for value in ("b200", "auto", ""):
        out = _run(value)
        assert out.returncode == 0, out.stderr
        assert out.stdout.strip() == "b200"


def test_invalid_env_flag_rejected():
    for value in ("numba", "fortran"):
        out = _run(value)
        assert out.returncode != 0
        assert "MTNN_BACKEND" in out.stderr


def test_active_backend_reports():
    assert kernels.active_backend() == "b200"


def test_missing_library_fails_loudly(tmp_path):
    env = dict(os.environ, MTNN_B200_LIB=str(tmp_path / "nope.so"), PYTHONPATH=str(ROOT))
    out = subprocess.run([sys.executable, "-c", "import paper_1702_03192_b200"],
                         capture_output=True, text=True, env=env, cwd=str(ROOT))
    assert out.returncode != 0 and "no CPU fallback" in out.stderr
