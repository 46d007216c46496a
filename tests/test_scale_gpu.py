"""BASELINE.json full-size configurations on the B200, checked through
properties that do not need a full float64 product: sampled float64 rows
(oracle_nt_rows), transpose involution and bit equality, NT == TNN agreement,
and empty / degenerate shapes."""

import numpy as np
import pytest

import oracle
from paper_1702_03192_b200 import device, kernels

pytestmark = pytest.mark.gpu
FP32_GATE = 1e-5


def _rand(shape, seed):
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.rand(shape, device="cuda", generator=g).mul_(2).sub_(1)


def _sampled_check(a, b, c, rows):
    """float64 dot products of sampled rows of C against all of B."""
    a_rows = a[rows].cpu().numpy()
    b_host = b.cpu().numpy()
    want = oracle.oracle_nt_rows(a_rows, b_host, np.arange(len(rows)), np.arange(b_host.shape[0]))
    got = c[rows].cpu().numpy()
    return oracle.rel_frobenius(got, want)


def test_config5_large_nt_65536x8192x8192():
    m, n, k = 65536, 8192, 8192
    a, b = _rand((m, k), 1), _rand((n, k), 2)
    c = device.gemm_nt(a, b)
    rows = np.sort(np.random.default_rng(0).choice(m, 32, replace=False))
    assert _sampled_check(a, b, c, rows) < FP32_GATE


@pytest.mark.parametrize("variant", ["tc3xf16s", "tc3xtf32"])
def test_sweep_max_case_16384_cubed_nt_equals_tnn(variant):
    import torch

    m = n = k = 16384
    a, b = _rand((m, k), 3), _rand((n, k), 4)
    code = {"tc3xf16s": 3, "tc3xtf32": 1}[variant]
    c_nt = device.gemm_nt(a, b, variant=code)
    rows = np.sort(np.random.default_rng(1).choice(m, 16, replace=False))
    assert _sampled_check(a, b, c_nt, rows) < FP32_GATE
    c_tnn = device.gemm_tnn(a, b, variant=code)
    # the two paths compute the same products in the same k order per chunk
    rel = float((c_tnn - c_nt).norm() / c_nt.norm())
    assert rel < 1e-6
    del c_tnn
    torch.cuda.empty_cache()


def test_transpose_16384_squared_bitexact_and_involution():
    import torch

    b = torch.randint(-2**31, 2**31 - 1, (16384, 16384), dtype=torch.int32,
                      device="cuda").view(torch.float32)
    bt = device.transpose(b)
    assert torch.equal(bt.view(torch.int32), b.view(torch.int32).t().contiguous())
    assert torch.equal(device.transpose(bt).view(torch.int32), b.view(torch.int32))


@pytest.mark.parametrize("shape", [(16384, 128), (128, 16384), (12345, 6789), (8191, 8193),
                                   (4097, 1023), (3000, 5000), (1, 100000), (100000, 1)])
def test_transpose_sweep_shapes_bitexact(shape):
    import torch

    b = torch.randint(-2**31, 2**31 - 1, shape, dtype=torch.int32, device="cuda").view(torch.float32)
    assert torch.equal(device.transpose(b).view(torch.int32), b.view(torch.int32).t().contiguous())


@pytest.mark.parametrize("m,n,k", [(0, 5, 3), (4, 0, 3), (4, 5, 0), (0, 0, 0)])
def test_empty_shapes(m, n, k):
    """Empty operands give empty / zero results on every path (the reference's
    numba loops do the same)."""
    import torch

    a = np.zeros((m, k), np.float32)
    b = np.zeros((n, k), np.float32)
    for fn in (kernels.gemm_nt, kernels.gemm_tnn):
        c = fn(a, b)
        assert c.shape == (m, n) and not c.any()
    c = kernels.gemm_nn(a, np.zeros((k, n), np.float32))
    assert c.shape == (m, n) and not c.any()
    assert kernels.transpose_oop(b).shape == (k, n)
    ta, tb = torch.zeros((m, k), device="cuda"), torch.zeros((n, k), device="cuda")
    tc = kernels.gemm_nt(ta, tb)
    assert tuple(tc.shape) == (m, n) and not tc.any()


def test_k_zero_gives_zeros_even_with_garbage_output():
    import torch

    a, b = torch.empty((64, 0), device="cuda"), torch.empty((32, 0), device="cuda")
    out = torch.full((64, 32), float("nan"), device="cuda")
    device.gemm_nt(a, b, out=out)
    assert torch.count_nonzero(out) == 0
