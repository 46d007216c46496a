"""Selector decisions (Algorithm 2) on the host, against the reference's
Dispatcher.select / gbdt.predict outputs (tests/golden/selector.npz).
Mirrors /root/reference/pkg/tests/test_selector.py where no GPU is needed
(free memory is passed explicitly)."""

import math
import time

import numpy as np
import pytest

from conftest import golden_model_names, golden_model_text
from paper_1702_03192_b200 import ProblemShape, gbdt, selector
from paper_1702_03192_b200.selector import (Choice, Dispatcher, Reason, SelectionDecision,
                                            build_features, select)

AMPLE = 1 << 40


def model(name):
    return gbdt.deserialize_model(golden_model_text(name))


def test_reference_row_vector(platform_a):
    got = build_features(platform_a, ProblemShape(128, 128, 128))
    assert got.tolist() == [8, 20, 1607, 256, 2048, 128, 128, 128]
    base = build_features(platform_a, ProblemShape(1, 2, 3))
    assert base[5:].tolist() == [1, 2, 3]


@pytest.mark.parametrize("name", golden_model_names())
def test_dispatcher_select_matches_reference(name, golden_selector, platform_a):
    g = golden_selector
    d = Dispatcher(model(name), platform_a)
    for sh, fr, ch, rs, raw in zip(g[f"{name}/shapes"], g[f"{name}/free"], g[f"{name}/choice"],
                                   g[f"{name}/reason"], g[f"{name}/sel_raw"]):
        dec = d.select(ProblemShape(*(int(v) for v in sh)), int(fr))
        assert (dec.choice is Choice.USE_TNN) == bool(ch)
        assert (dec.reason is Reason.MEMORY_FALLBACK) == bool(rs)
        if rs:
            assert math.isnan(dec.raw_score)
        else:
            assert dec.raw_score == raw


@pytest.mark.parametrize("name", golden_model_names())
def test_decision_agrees_with_learner_predict(name, golden_selector, platform_a):
    g = golden_selector
    m = model(name)
    d = Dispatcher(m, platform_a)
    for x, lab in zip(g[f"{name}/x"], g[f"{name}/label"]):
        if not float(x[5]).is_integer() or not float(x[7]).is_integer():
            continue  # shapes are integers; float probes are covered by the walkers
        shape = ProblemShape(int(x[5]), int(x[6]), int(x[7]))
        dec = d.select(shape, AMPLE)
        assert (dec.choice is Choice.USE_NT) == (lab == 1)
        one_shot = select(m, platform_a, shape, AMPLE)
        assert one_shot.choice is dec.choice and one_shot.raw_score == dec.raw_score


def test_memory_fallback(platform_a):
    d = Dispatcher(model("const_neg"), platform_a)
    dec = d.select(ProblemShape(1, 1, 1), free_memory=0)
    assert dec.choice is Choice.USE_NT and dec.reason is Reason.MEMORY_FALLBACK
    assert math.isnan(dec.raw_score)
    dec = select(model("const_neg"), platform_a, ProblemShape(1, 1, 1), free_memory=0)
    assert dec.reason is Reason.MEMORY_FALLBACK and math.isnan(dec.raw_score)
    # exactly enough memory -> the model decides (4*n*k <= free)
    dec = d.select(ProblemShape(8, 8, 8), free_memory=4 * 8 * 8)
    assert dec.reason is Reason.PREDICTED and dec.choice is Choice.USE_TNN


def test_never_tnn_without_memory(platform_a, rng):
    d = Dispatcher(model("const_neg"), platform_a)
    for _ in range(200):
        shape = ProblemShape(*(int(v) for v in rng.integers(1, 4096, 3)))
        budget = int(rng.integers(0, 4 * shape.n * shape.k))
        dec = d.select(shape, budget)
        if 4 * shape.n * shape.k > budget:
            assert dec.choice is Choice.USE_NT and dec.reason is Reason.MEMORY_FALLBACK


def test_fallback_decision_invariant():
    with pytest.raises(ValueError, match="fallback"):
        SelectionDecision(Choice.USE_TNN, Reason.MEMORY_FALLBACK, 0.0)


def test_empty_model_dispatches_nt(platform_a):
    m = gbdt.GbdtModel(trees=(), params=gbdt.GbdtParams(), n_features=8)
    dec = Dispatcher(m, platform_a).select(ProblemShape(8, 8, 8), AMPLE)
    assert dec.choice is Choice.USE_NT and dec.raw_score == 0.0


def test_wrong_arity_model_rejected(platform_a):
    m = gbdt.GbdtModel(trees=(gbdt.TreeNode(weight=1.0),), params=gbdt.GbdtParams(), n_features=3)
    with pytest.raises(ValueError, match="8 features"):
        Dispatcher(m, platform_a)


def test_selection_overhead_budget(platform_a):
    # reference budget: median <= 100 us (test_selector.py:179-200); the
    # native walk makes the Python-visible select a few microseconds
    d = Dispatcher(model("size_rule"), platform_a)
    shape = ProblemShape(512, 512, 512)
    d.select(shape, AMPLE)
    samples = []
    for _ in range(500):
        t0 = time.perf_counter()
        d.select(shape, AMPLE)
        samples.append(time.perf_counter() - t0)
    assert float(np.median(samples)) <= 1e-4


def test_native_decision_is_sub_microsecond(platform_a):
    """The host C++ evaluator itself (excluding the Python call) is < 1 us."""
    import ctypes

    from paper_1702_03192_b200 import _lib

    native = gbdt.NativeModel.from_json(golden_model_text("fixture"))
    prefix = np.array(platform_a.as_tuple())
    p = prefix.ctypes.data_as(_lib._DP)
    raw, ch, rs = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
    n, batches = 4000, []
    for _ in range(5):  # best batch: robust to other load on the host
        t0 = time.perf_counter()
        for i in range(n):
            _lib.lib.mtnn_select(native.handle, p, 512, 512, 512, AMPLE, ctypes.byref(raw),
                                 ctypes.byref(ch), ctypes.byref(rs))
        batches.append((time.perf_counter() - t0) / n)
    per_call = min(batches)
    # the ctypes round trip dominates (~1.4 us idle); the measured total bounds the
    # native cost. Loose bound (a loaded CI host); the FFI-free test below pins
    # the evaluator itself. Reference select(): 10.5 us.
    assert per_call < 1e-5


def test_native_decision_cost_without_ffi(platform_a):
    """mtnn_select in C++ alone (no ctypes round trip) is sub-microsecond."""
    import ctypes

    from paper_1702_03192_b200 import _lib

    native = gbdt.NativeModel.from_json(golden_model_text("fixture"))
    prefix = np.array(platform_a.as_tuple())
    ns = ctypes.c_double()
    _lib.check(_lib.lib.mtnn_select_cost_ns(native.handle, prefix.ctypes.data_as(_lib._DP),
                                            200000, ctypes.byref(ns)))
    assert 0 < ns.value < 1000.0, ns.value
