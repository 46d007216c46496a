"""The C-ABI library loads without a GPU and exports exactly what
include/mtnn_b200.h declares; host-only entry points (model, selector, tree
walkers) are exercised here against the reference's golden outputs."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden_model_names, golden_model_text
from paper_1702_03192_b200 import _lib, gbdt
from paper_1702_03192_b200.kernels import _b200_impl

HEADER = ROOT / "include" / "mtnn_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mtnn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_abi_version_and_error_plumbing():
    assert _lib.lib.mtnn_abi_version() == 1
    # unknown variant -> EINVAL -> ValueError, message in mtnn_last_error
    rc = _lib.lib.mtnn_gemm_nt(None, None, None, -1, 1, 1, 0, None)
    assert rc == _lib.EINVAL
    with pytest.raises(ValueError, match="non-negative"):
        _lib.check(rc)


def test_no_gpu_is_reported_not_faked():
    if _lib.lib.mtnn_device_available():
        pytest.skip("a GPU is present")
    a = np.ones((4, 4), np.float32)
    c = np.empty((4, 4), np.float32)
    rc = _lib.lib.mtnn_gemm_nt_host(a.ctypes.data, a.ctypes.data, c.ctypes.data, 4, 4, 4, 0)
    assert rc == _lib.ENOTSUP
    assert "device" in _lib.last_error().lower() or "cuda" in _lib.last_error().lower()


@pytest.mark.parametrize("name", golden_model_names())
def test_json_model_matches_reference_predict(name, golden_selector):
    g = golden_selector
    native = gbdt.NativeModel.from_json(golden_model_text(name))
    for v, r in zip(g[f"{name}/x"], g[f"{name}/raw"]):
        assert native.raw(v) == r  # bit-identical float64


@pytest.mark.parametrize("name", golden_model_names())
def test_packed_walkers_match_reference(name, golden_selector):
    g = golden_selector
    packed = [g[f"{name}/{f}"] for f in ("feat", "thresh", "left", "right", "leaf")]
    base, eta = g[f"{name}/base"]
    for v, r in zip(g[f"{name}/x"][:200], g[f"{name}/raw"][:200]):
        assert _b200_impl.walk_trees(*packed, v, base, eta) == r
        assert _b200_impl.walk_trees_mnk(*packed, v[:5], v[5], v[6], v[7], base, eta) == r


@pytest.mark.parametrize("name", golden_model_names())
def test_python_model_roundtrip_and_pack(name, golden_selector):
    g = golden_selector
    text = golden_model_text(name)
    model = gbdt.deserialize_model(text)
    assert gbdt.serialize_model(model) == text  # byte-identical wire format
    for got, key in zip(gbdt.pack_trees(model), ("feat", "thresh", "left", "right", "leaf")):
        assert np.array_equal(got, g[f"{name}/{key}"])
    for v, r, lab in zip(g[f"{name}/x"][:300], g[f"{name}/raw"][:300], g[f"{name}/label"][:300]):
        assert gbdt.predict_raw(model, v) == r
        assert gbdt.predict(model, v) == lab


@pytest.mark.parametrize("doc, msg", [
    ("not json", "not valid JSON"),
    ("[]", "expected a JSON object"),
    ('{"version": 1}', "missing 'params'"),
    ('{"version": 2, "params": {}, "base_score": 0, "trees": []}', "unsupported version"),
    ('{"version": 1, "params": {"max_depth": 8}, "base_score": 0, "trees": []}', "missing 'n_estimators'"),
    ('{"version": 1, "params": {"max_depth": 8, "n_estimators": 1, "eta": 1, "gamma": 0, "lambda": 1,'
     ' "min_child_weight": 1}, "base_score": 0, "trees": [{"feat": -1, "thresh": 0, "left": {"leaf": 0},'
     ' "right": {"leaf": 0}}]}', "feat"),
    ('{"version": 1, "params": {"max_depth": 8, "n_estimators": 1, "eta": 1, "gamma": 0, "lambda": 1,'
     ' "min_child_weight": 1}, "base_score": 0, "trees": [{"leaf": 0}, {"leaf": 1}]}', "exceeds n_estimators"),
    ('{"version": 1, "params": {"max_depth": 8, "n_estimators": 1, "eta": 1, "gamma": 0, "lambda": 1,'
     ' "min_child_weight": 1}, "base_score": 0, "trees": [{"feat": 0, "thresh": 0, "left": {"leaf": 0}}]}',
     "missing 'right'"),
])
def test_malformed_documents_rejected_by_both_readers(doc, msg):
    with pytest.raises(gbdt.ModelFormatError, match=msg):
        gbdt.NativeModel.from_json(doc)
    with pytest.raises(gbdt.ModelFormatError):
        gbdt.deserialize_model(doc)


def test_native_raw_validates_like_predict_raw():
    native = gbdt.NativeModel.from_json(golden_model_text("size_rule"))
    with pytest.raises(ValueError, match="8 features"):
        native.raw(np.zeros(7))
    with pytest.raises(ValueError, match="finite"):
        native.raw(np.array([1, 1, 1, 1, 1, np.nan, 1, 1.0]))


def test_config_knobs_roundtrip_and_reject_unknown():
    key = "f16s_inkernel_max_short"
    old = _lib.config_get(key)
    try:
        _lib.config_set(key, 0)
        assert _lib.config_get(key) == 0
        _lib.config_set(key, 256)
        assert _lib.config_get(key) == 256
        with pytest.raises(ValueError, match=">= 0"):
            _lib.config_set(key, -1)
    finally:
        _lib.config_set(key, old)
    with pytest.raises(ValueError, match="unknown config key"):
        _lib.config_set("no_such_knob", 1)
    old = _lib.config_get("host_pipeline_zc")
    try:
        for v in (1, 0):
            _lib.config_set("host_pipeline_zc", v)
            assert _lib.config_get("host_pipeline_zc") == v
        with pytest.raises(ValueError):
            _lib.config_set("host_pipeline_zc", 2)
    finally:
        _lib.config_set("host_pipeline_zc", old)



def test_ipc_and_allgather_fail_cleanly_without_a_gpu():
    """The multi-GPU entry points report errors (no crash) on bad input / no GPU."""
    import ctypes

    lib = _lib.lib
    h = (ctypes.c_char * 64)()
    off = ctypes.c_int64()
    assert lib.mtnn_ipc_handle(None, ctypes.addressof(h), ctypes.byref(off)) == _lib.EINVAL
    p = ctypes.c_void_p()
    assert lib.mtnn_ipc_open(None, 0, ctypes.byref(p)) == _lib.EINVAL
    assert lib.mtnn_ipc_close(ctypes.c_void_p(1234)) == _lib.EINVAL
    assert "not opened" in _lib.last_error()
    rc = lib.mtnn_gemm_nt_allgather(None, None, None, None, 0, -1, 4, 4, 4, None)
    assert rc == _lib.EINVAL and "row0" in _lib.last_error()
    rc = lib.mtnn_gemm_nt_allgather(None, None, None, None, 2, 0, 4, 4, 4, None)
    assert rc == _lib.EINVAL and "peer" in _lib.last_error()
    if not lib.mtnn_device_available():
        buf = (ctypes.c_float * 16)()
        assert lib.mtnn_ipc_handle(ctypes.addressof(buf), ctypes.addressof(h), ctypes.byref(off)) != 0
