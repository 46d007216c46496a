"""The in-package learner (paper_1702_03192_b200.learn) trains the same
models and CV reports as the reference's fit_gbdt / cross_validate
(gbdt.py:207-350) — pinned by tests/golden/learn.npz, which
tests/golden/make_golden_learn.py wrote by running the reference."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1702_03192_b200 import gbdt, learn

PARAMS = {
    "default": gbdt.GbdtParams(),
    "squared": gbdt.GbdtParams(max_depth=4, n_estimators=3, eta=0.3, objective="squared"),
    "regularised": gbdt.GbdtParams(max_depth=5, n_estimators=6, eta=0.5, gamma=0.1, lam=2.0,
                                   min_child_weight=3.0),
}
SETS = ("fixture", "noisy_rule", "continuous")


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(GOLDEN / "learn.npz"))


@pytest.mark.parametrize("sname", SETS)
@pytest.mark.parametrize("pname", sorted(PARAMS))
def test_fit_gbdt_matches_reference_model(golden, sname, pname):
    x, y = golden[f"{sname}/x"], golden[f"{sname}/y"]
    model = learn.fit_gbdt(x, y, PARAMS[pname])
    assert gbdt.serialize_model(model) == str(golden[f"{sname}/{pname}/model"])


@pytest.mark.parametrize("sname", SETS)
@pytest.mark.parametrize("pname", sorted(PARAMS))
def test_cross_validate_matches_reference(golden, sname, pname):
    x, y = golden[f"{sname}/x"], golden[f"{sname}/y"]
    cv = learn.cross_validate(x, y, folds=5, params=PARAMS[pname], seed=3)
    want = json.loads(str(golden[f"{sname}/{pname}/cv"]))
    got = [list(cv.fold_accuracies), list(cv.negative), list(cv.positive), list(cv.total)]
    assert json.dumps(got) == json.dumps(want)


def test_learner_validation():
    with pytest.raises(ValueError, match="empty"):
        learn.fit_gbdt(np.zeros((0, 8)), np.zeros(0))
    with pytest.raises(ValueError, match="-1 or \\+1"):
        learn.fit_gbdt(np.zeros((3, 8)), np.array([0, 1, 1]))
    with pytest.raises(ValueError, match="folds"):
        learn.cross_validate(np.zeros((3, 8)), np.ones(3), folds=1)
    with pytest.raises(ValueError, match="finite"):
        learn.fit_tree(np.zeros((2, 8)), np.array([np.nan, 0.0]), np.ones(2))


def test_constant_labels_give_single_leaf_trees():
    x = np.random.default_rng(0).uniform(size=(20, 8))
    model = learn.fit_gbdt(x, np.full(20, -1))
    assert all(t.is_leaf for t in model.trees)
    assert gbdt.predict(model, x[0]) == -1
