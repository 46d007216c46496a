"""Device operand generator vs the reference harness's make_operands
(pkg/src/mtnn/bench.py:104-114): bit-identical float32 values."""

import numpy as np
import pytest
import torch

import oracle
from paper_1702_03192_b200 import operands

pytestmark = pytest.mark.gpu


def test_golden_make_operands(golden_operands):
    g = golden_operands
    for i in range(3):
        m, n, k, seed = (int(x) for x in g[f"shape{i}"])
        a, b = operands.make_operands(m, n, k, seed)
        assert np.array_equal(a.cpu().numpy(), g[f"a{i}"])
        assert np.array_equal(b.cpu().numpy(), g[f"b{i}"])


@pytest.mark.parametrize("count,skip,seed", [(1, 0, 0), (31, 0, 0), (33, 5, 1), (4097, 12345, 7),
                                             (1 << 20, 3, 0), (300001, (1 << 33) + 17, 42)])
def test_stream_matches_numpy(count, skip, seed):
    rng = np.random.default_rng(seed)
    if skip:
        rng.bit_generator.advance(skip)
    want = rng.uniform(-1.0, 1.0, count).astype(np.float32)
    got = torch.empty(count, dtype=torch.float32, device="cuda")
    operands.fill_uniform(got, seed, skip)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("shape", [(128, 256, 512), (1000, 3, 77), (4096, 4096, 64)])
def test_shapes_and_views(shape):
    m, n, k = shape
    a_ref, b_ref, _ = oracle.make_operands(m, n, k, 0)
    a, b = operands.make_operands(m, n, k, 0)
    assert np.array_equal(a.cpu().numpy(), a_ref) and np.array_equal(b.cpu().numpy(), b_ref)
    stream = operands.operand_stream(2 * 4096 * 4096, 0)
    av, bv = operands.views(stream, m, n, k)
    assert torch.equal(av, a) and torch.equal(bv, b)
