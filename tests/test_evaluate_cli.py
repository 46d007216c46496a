"""Evaluation layer (GOW/LUB report) and CLI: parity with the reference's
metrics.aggregate / render_report and its CSV wire formats (tests/golden/)."""

import csv
import io

import numpy as np
import pytest

from conftest import GOLDEN, PLATFORM_A, golden_model_text
from paper_1702_03192_b200 import cli, evaluate, gbdt, sweep
from paper_1702_03192_b200.kernels import ProblemShape
from paper_1702_03192_b200.platform import PlatformFeatures
from paper_1702_03192_b200.selector import Dispatcher


@pytest.fixture(scope="module")
def golden_eval():
    return dict(np.load(GOLDEN / "evaluate.npz"))


@pytest.mark.parametrize("i,mode", [(0, "remeasured"), (1, "copied")])
def test_aggregate_matches_reference(golden_eval, i, mode):
    p = golden_eval[f"p{i}"]
    cases = [evaluate.EvalCase(ProblemShape(1, 1, 1), a, b, c) for a, b, c in p]
    rep = evaluate.aggregate(cases, p_mtnn_mode=mode)
    got = [rep.mtnn_vs_nt, rep.mtnn_vs_tnn, rep.gow_avg, rep.gow_max, rep.lub_avg, rep.lub_min]
    np.testing.assert_allclose(got, golden_eval[f"vals{i}"], rtol=1e-12, atol=1e-12)
    assert list(rep.ratio_histogram) == list(golden_eval[f"hist{i}"])
    assert evaluate.render_report(rep) + "\n" == (GOLDEN / f"report{i}.txt").read_text()


def test_metric_definitions():
    assert evaluate.gow(3.0, 1.0, 2.0) == 2.0
    assert evaluate.lub(1.0, 1.0, 2.0) == -0.5
    assert evaluate.ratio_histogram([0.0, 0.05, 0.1, 1.99, 2.0, 7.5]) == (
        2, 1) + (0,) * 17 + (1, 2)
    with pytest.raises(ValueError):
        evaluate.gow(0.0, 1.0, 1.0)
    with pytest.raises(ValueError, match="no cases"):
        evaluate.aggregate([])


def _timing_rows():
    return sweep.rows_from_timings(sweep.read_timings_csv(GOLDEN / "wire_t.csv"))


def test_records_and_samples_wire_format(tmp_path):
    plat = PlatformFeatures(**{k: float(v) for k, v in PLATFORM_A.items()})
    rows = _timing_rows()
    sweep.write_records_csv(tmp_path / "r.csv", rows)
    sweep.write_samples_csv(tmp_path / "s.csv", rows, plat)
    assert (tmp_path / "r.csv").read_text() == (GOLDEN / "wire_r.csv").read_text()
    assert (tmp_path / "s.csv").read_text() == (GOLDEN / "wire_s.csv").read_text()


def test_evaluate_injected_copied_mode():
    plat = PlatformFeatures(**{k: float(v) for k, v in PLATFORM_A.items()})
    d = Dispatcher(gbdt.deserialize_model(golden_model_text("fixture")), plat)
    timings = sweep.read_timings_csv(GOLDEN / "wire_t.csv")
    shapes = [ProblemShape(*s) for s in timings]
    cases = evaluate.evaluate_cases(d, shapes, injected=timings)
    for c in cases:
        assert c.p_mtnn in (c.p_nt, c.p_tnn)
        assert evaluate.gow(c.p_mtnn, c.p_nt, c.p_tnn) >= 0
        assert evaluate.lub(c.p_mtnn, c.p_nt, c.p_tnn) <= 0
    with pytest.raises(KeyError, match="missing case"):
        evaluate.evaluate_cases(d, [ProblemShape(3, 3, 3)], injected=timings)


OVR = [f"--platform-override={k}={v}" for k, v in PLATFORM_A.items()]


def test_cli_sweep_inject_eval_predict(tmp_path, capsys):
    model = tmp_path / "m.json"
    model.write_text(golden_model_text("fixture"))
    rc = cli.main(["sweep", "--exp-min", "5", "--exp-max", "7", "--inject", str(GOLDEN / "wire_t.csv"),
                   "--records", str(tmp_path / "r.csv"), "--samples", str(tmp_path / "s.csv"), *OVR])
    assert rc == 0
    assert (tmp_path / "s.csv").read_text() == (GOLDEN / "wire_s.csv").read_text()
    rc = cli.main(["eval", "--model", str(model), "--exp-min", "5", "--exp-max", "7",
                   "--inject", str(GOLDEN / "wire_t.csv"), "--out", str(tmp_path / "rep.csv"),
                   "--hist-out", str(tmp_path / "h.csv"), *OVR])
    assert rc == 0
    rows = list(csv.reader(open(tmp_path / "rep.csv")))
    assert rows[0] == ["metric", "percent"] and rows[-2] == ["p_mtnn_mode", "copied"]
    rc = cli.main(["predict", "--model", str(model), "--free-memory", str(1 << 40), *OVR, "64", "64", "64"])
    assert rc == 0
    out = capsys.readouterr().out
    assert out.strip().splitlines()[-1].split()[0] in ("NT", "TNN")
    rc = cli.main(["predict", "--model", str(model), "--free-memory", "0", *OVR, "64", "64", "64"])
    assert "memory_fallback" in capsys.readouterr().out


def test_cli_errors_exit_1(tmp_path, capsys):
    rc = cli.main(["predict", "--model", str(tmp_path / "missing.json"), *OVR, "1", "1", "1"])
    assert rc == 1 and "error:" in capsys.readouterr().err


def test_cli_train_and_cv(tmp_path, capsys):
    model = tmp_path / "m.json"
    rc = cli.main(["train", "--samples", str(GOLDEN / "wire_s.csv"), "--model", str(model)])
    assert rc == 0 and model.exists()
    gbdt.load_model(model)  # loads with this package's reader
    rc = cli.main(["cv", "--samples", str(GOLDEN / "wire_s.csv"), "--folds", "3"])
    assert rc == 0 and "Total" in capsys.readouterr().out


@pytest.mark.gpu
def test_evaluate_remeasured_on_gpu():
    from paper_1702_03192_b200.platform import probe_platform

    d = Dispatcher(gbdt.deserialize_model(golden_model_text("const_pos")), probe_platform())
    shapes = [ProblemShape(*s) for s in sweep.grid_shapes(range(7, 9))]
    cases = evaluate.evaluate_cases(d, shapes, reps=3, warmup=1)
    rep = evaluate.aggregate(cases)
    assert rep.n_cases == 8 and all(c.p_nt > 0 and c.p_tnn > 0 and c.p_mtnn > 0 for c in cases)


@pytest.mark.gpu
def test_cli_demo_fcn_and_sweep_on_gpu(tmp_path, capsys):
    model = tmp_path / "m.json"
    model.write_text(golden_model_text("const_pos"))
    assert cli.main(["demo-fcn", "--model", str(model), "--iters", "1", "--batch", "8"]) == 0
    out = capsys.readouterr().out
    assert "Total" in out and "NT/MTNN" in out
    assert cli.main(["sweep", "--exp-min", "7", "--exp-max", "8", "--reps", "2", "--warmup", "1",
                     "--records", str(tmp_path / "r.csv"), "--samples", str(tmp_path / "s.csv"),
                     "--timings", str(tmp_path / "t.csv")]) == 0
    assert len(open(tmp_path / "s.csv").read().splitlines()) == 9


def test_lpt_shards_balance():
    shapes = sweep.grid_shapes(range(7, 12))
    owner = sweep.lpt_shards(shapes, 4)
    loads = [sum(m * n * k for (m, n, k), o in zip(shapes, owner) if o == r) for r in range(4)]
    assert set(owner) == {0, 1, 2, 3} and max(loads) / min(loads) < 1.05


def test_cli_device_flags_parse():
    p = cli.build_parser()
    a = p.parse_args(["sweep", "--device", "1", "--gpus", "4", "--threads", "8", "--block", "64",
                      "--tile", "16"])
    assert (a.device, a.gpus, a.threads) == (1, 4, 8)
    a = p.parse_args(["eval", "--gpus", "2"])
    assert a.gpus == 2 and a.device == 0
    assert p.parse_args(["predict", "--device", "3", "1", "2", "3"]).device == 3


@pytest.mark.gpu
def test_cases_sharded_over_processes_on_gpu():
    """The --gpus path (one process per GPU, LPT shards, results in grid order),
    exercised with two processes on GPU 0."""
    shapes = sweep.grid_shapes(range(7, 9))
    rows = sweep.map_cases_on_gpus(sweep._sweep_worker, shapes, 2, (2, 1, 0), devices=[0, 0])
    assert [(r.m, r.n, r.k) for r in rows] == [tuple(s) for s in shapes]
    assert all(r.t_nt > 0 and r.t_tnn > 0 and r.t_nn > 0 for r in rows)
    from paper_1702_03192_b200.platform import probe_platform

    d = Dispatcher(gbdt.deserialize_model(golden_model_text("const_pos")), probe_platform())
    cases = sweep.map_cases_on_gpus(evaluate._eval_worker, [tuple(s) for s in shapes], 2,
                                    (gbdt.serialize_model(d.model), tuple(d.platform.as_tuple()),
                                     2, 1, "remeasured"), devices=[0, 0])
    assert [tuple(c.shape) for c in cases] == [tuple(s) for s in shapes]
