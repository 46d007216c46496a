"""FCN workload (config 4): mirrors /root/reference/pkg/tests/test_fcn.py."""

import numpy as np
import pytest

from conftest import golden_model_text
from paper_1702_03192_b200 import fcn, gbdt
from paper_1702_03192_b200.fcn import (DEFAULT_BATCHES, FcnInfeasibleError, compare_dispatchers,
                                       fcn_scenario, iteration_flops, preset_widths,
                                       scaled_widths)
from paper_1702_03192_b200.selector import Dispatcher


class TestPresets:
    def test_mnist_like_widths(self):
        assert preset_widths("mnist-like", 2) == (784, 10, (2048, 1024))
        assert preset_widths("mnist-like", 4) == (784, 10, (2048, 2048, 2048, 1024))

    def test_synthetic_like_widths(self):
        in_dim, out_dim, hidden = preset_widths("synthetic-like", 3)
        assert in_dim == out_dim == 26752 and hidden == (4096, 4096, 4096)

    def test_unknown_preset(self):
        with pytest.raises(ValueError, match="unknown preset"):
            preset_widths("imagenet", 2)

    def test_unsupported_depth(self):
        with pytest.raises(ValueError, match="hidden layers"):
            preset_widths("mnist-like", 5)

    def test_scaled_widths(self):
        assert scaled_widths((26752, 4096), 8) == (3344, 512)
        assert scaled_widths((10,), 16) == (1,)
        with pytest.raises(ValueError, match="divisor"):
            scaled_widths((8,), 0)

    def test_default_batches_cover_presets(self):
        assert set(DEFAULT_BATCHES) == set(fcn.PRESETS)

    def test_config4_flops(self):
        # BASELINE config 4: 784-4096-4096-4096-10, batch 1024 -> 2.2614e11 flop/step
        assert iteration_flops((4096,) * 3, 1024, 784, 10) == 6 * 1024 * (784 * 4096 + 2 * 4096 * 4096 + 4096 * 10)  # 2.2614e11


class TestValidation:
    def test_invalid_dispatch(self):
        with pytest.raises(ValueError, match="dispatch"):
            fcn_scenario([4], 2, 3, 2, "cublas")

    def test_invalid_iters(self):
        with pytest.raises(ValueError, match="iters"):
            fcn_scenario([4], 2, 3, 2, "nt", iters=0)
        with pytest.raises(ValueError, match="iters"):
            compare_dispatchers({"nt": "nt"}, [4], (2,), 3, 2, iters=0)

    def test_invalid_backward_mode(self):
        with pytest.raises(ValueError, match="backward_nt"):
            fcn_scenario([4], 2, 3, 2, "nt", backward_nt="maybe")


@pytest.mark.gpu
class TestScenarioGpu:
    def test_smallest_network_runs(self):
        r = fcn_scenario([1], batch=1, input_dim=1, output_dim=1, dispatch="nt")
        assert r.forward_seconds > 0 and r.backward_seconds > 0
        assert r.total_seconds == pytest.approx(r.forward_seconds + r.backward_seconds)

    def test_call_log_shapes(self):
        r = fcn_scenario([6], batch=4, input_dim=5, output_dim=3, dispatch="nt")
        fwd = [c for c in r.calls if c.phase == "forward"]
        bwd = [c for c in r.calls if c.phase == "backward"]
        assert [(c.op, c.m, c.n, c.k) for c in fwd] == [("nt", 4, 6, 5), ("nt", 4, 3, 6)]
        assert [(c.op, c.m, c.n, c.k) for c in bwd] == [
            ("nn", 4, 6, 3), ("nt-fixed", 3, 6, 4), ("nn", 4, 5, 6), ("nt-fixed", 6, 5, 4)]
        assert all(c.seconds >= 0 for c in r.calls)

    def test_all_nt_dispatched(self, platform_a):
        d = Dispatcher(gbdt.deserialize_model(golden_model_text("const_pos")), platform_a)
        r = fcn_scenario([6], 4, 5, 3, d, backward_nt="dispatch")
        assert [c.op for c in r.calls if c.phase == "backward"] == ["nn", "nt", "nn", "nt"]

    def test_dispatch_modes(self, platform_a):
        d = Dispatcher(gbdt.deserialize_model(golden_model_text("size_rule")), platform_a)
        for dispatch in ("nt", "tnn", d):
            assert fcn_scenario([4], 2, 3, 2, dispatch).forward_seconds > 0

    def test_invalid_sizes(self):
        with pytest.raises(ValueError, match="batch"):
            fcn_scenario([4], 0, 3, 2, "nt")
        with pytest.raises(ValueError, match="widths"):
            fcn_scenario([0], 2, 3, 2, "nt")

    def test_infeasible_names_layer(self):
        with pytest.raises(FcnInfeasibleError, match="layer 1"):
            fcn_scenario([2, 200_000], batch=200_000, input_dim=2, output_dim=200_000,
                         dispatch="nt", mem_fraction=0.05)

    def test_compare_dispatchers(self, platform_a):
        d = Dispatcher(gbdt.deserialize_model(golden_model_text("size_rule")), platform_a)
        totals = compare_dispatchers({"nt": "nt", "tnn": "tnn", "mtnn": d}, hidden=[64, 64],
                                     batches=(32, 64), input_dim=64, output_dim=64, iters=2)
        assert set(totals) == {"nt", "tnn", "mtnn"}
        for f, b in totals.values():
            assert f > 0 and b > 0

    def test_config4_results_match_oracle(self):
        """The forward products of config 4's layers are FP32-accurate."""
        import torch

        import oracle

        layers = fcn._build_layers((4096,) * 3, 1024, 784, 10, 0, 0.8, "cuda")
        for l in layers:
            got = fcn._nt_call("nt", l["x"], l["w"]).cpu().numpy()
            want = oracle.oracle_nt_blas(l["x"].cpu().numpy(), l["w"].cpu().numpy())
            assert oracle.rel_frobenius(got, want) < 1e-5
