"""Dispatcher.gemm on the GPU (mirrors reference tests/test_selector.py:112-156
and test_mtnn_gemm_convenience)."""

import logging

import numpy as np
import pytest

import oracle
from conftest import golden_model_text
from oracle import random_matrix, rel_frobenius
from paper_1702_03192_b200 import gbdt, selector
from paper_1702_03192_b200.selector import Choice, Dispatcher, mtnn_gemm

pytestmark = pytest.mark.gpu
AMPLE = 1 << 40


def model(name):
    return gbdt.deserialize_model(golden_model_text(name))


def test_gemm_matches_oracle(platform_a, rng):
    d = Dispatcher(model("size_rule"), platform_a)
    for _ in range(50):
        m, n, k = (int(v) for v in rng.integers(1, 48, 3))
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        assert rel_frobenius(d.gemm(a, b), oracle.oracle_nt(a, b)) < 1e-4


def test_gemm_identity(platform_a, rng):
    d = Dispatcher(model("size_rule"), platform_a)
    a = random_matrix(rng, 5, 5)
    assert rel_frobenius(d.gemm(a, np.eye(5, dtype=np.float32)), a) < 1e-6


def test_branches_agree(platform_a, rng):
    d_nt = Dispatcher(model("const_pos"), platform_a)
    d_tnn = Dispatcher(model("const_neg"), platform_a)
    worst = 0.0
    for _ in range(100):
        m, n, k = (int(v) for v in rng.integers(1, 40, 3))
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        worst = max(worst, rel_frobenius(d_tnn.gemm(a, b), d_nt.gemm(a, b)))
    assert worst <= 1e-4


def test_branches_agree_large_on_device(platform_a, rng):
    import torch

    d_nt = Dispatcher(model("const_pos"), platform_a)
    d_tnn = Dispatcher(model("const_neg"), platform_a)
    a, b = random_matrix(rng, 1024, 768), random_matrix(rng, 512, 768)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c1 = d_nt.gemm(ta, tb)
    assert d_nt.last_choice is Choice.USE_NT
    c2 = d_tnn.gemm(ta, tb)
    assert d_tnn.last_choice is Choice.USE_TNN
    want = oracle.oracle_nt_blas(a, b)
    assert rel_frobenius(c1.cpu().numpy(), want) < 1e-5
    assert rel_frobenius(c2.cpu().numpy(), want) < 1e-5
    # memory guard forces NT on the device path too
    d_tnn.gemm(ta, tb, free_memory=0)
    assert d_tnn.last_choice is Choice.USE_NT


def test_memory_error_retries_as_nt(platform_a, rng, monkeypatch, caplog):
    d = Dispatcher(model("const_neg"), platform_a)

    def boom(*args, **kwargs):
        raise MemoryError("no room")

    monkeypatch.setattr(selector._impl, "gemm_tnn", boom)
    a, b = random_matrix(rng, 4, 6), random_matrix(rng, 5, 6)
    with caplog.at_level(logging.WARNING, logger=selector.__name__):
        got = d.gemm(a, b, free_memory=AMPLE)
    assert rel_frobenius(got, oracle.oracle_nt(a, b)) < 1e-4
    assert any("retrying as NT" in rec.message for rec in caplog.records)


def test_gemm_validates_inputs(platform_a, rng):
    d = Dispatcher(model("const_pos"), platform_a)
    with pytest.raises(ValueError, match="share k"):
        d.gemm(random_matrix(rng, 2, 3), random_matrix(rng, 2, 4))
    with pytest.raises(TypeError, match="float32"):
        d.gemm(np.ones((2, 2)), random_matrix(rng, 2, 2))


def test_free_memory_is_device_memory(platform_a):
    free = selector._free_memory_bytes()
    assert free > 1 << 30


def test_mtnn_gemm_convenience(platform_a, rng):
    a, b = random_matrix(rng, 6, 4), random_matrix(rng, 5, 4)
    assert rel_frobenius(mtnn_gemm(model("const_pos"), platform_a, a, b),
                         oracle.oracle_nt(a, b)) < 1e-4


def test_probe_platform_reads_the_b200():
    from paper_1702_03192_b200.platform import probe_platform

    p = probe_platform()
    assert p.sm == 148 and p.gm > 170 and p.l2c > 100_000
