"""Golden fixtures for the selector learner (tests/test_learn.py).

Run in the build container, where the reference imports:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_learn.py
Writes tests/golden/learn.npz: training sets (features, labels), the model the
reference's fit_gbdt trains on each (serialize_model text) and its
cross_validate report, for default and non-default GbdtParams.
"""

import json
from pathlib import Path

import numpy as np
from mtnn import bench, gbdt
from mtnn.platform import PlatformFeatures

OUT = Path(__file__).resolve().parent / "learn.npz"


def main():
    rng = np.random.default_rng(20260417)
    plat = PlatformFeatures(gm=8.0, sm=20.0, cc=1607.0, mbw=256.0, l2c=2048.0)
    sets = {}
    # the reference pipeline on its deterministic fixture timings (grid 2^5..2^11)
    injected = {tuple(s): bench.synthetic_timings(s) for s in bench.grid_shapes(range(5, 12))}
    records = bench.sweep_grid(range(5, 12), plat, injected=injected)
    sets["fixture"] = bench.samples_to_arrays(bench.label_records(records, plat))
    # a size rule with label noise and repeated feature values (ties)
    n = 400
    x = np.column_stack([np.full(n, 180.0), np.full(n, 148.0), np.full(n, 1965.0),
                         np.full(n, 8192.0), np.full(n, 129024.0),
                         2.0 ** rng.integers(7, 15, n), 2.0 ** rng.integers(7, 15, n),
                         2.0 ** rng.integers(7, 15, n)])
    y = np.where(x[:, 5] * x[:, 6] * x[:, 7] < 2.0 ** 33, 1, -1)
    flip = rng.random(n) < 0.08
    y[flip] = -y[flip]
    sets["noisy_rule"] = (x, y)
    # continuous features, imbalanced classes
    x = rng.normal(size=(300, 8))
    y = np.where(x[:, 0] + 0.5 * x[:, 3] ** 2 > 1.2, -1, 1)
    sets["continuous"] = (x, y)
    params = {
        "default": gbdt.GbdtParams(),
        "squared": gbdt.GbdtParams(max_depth=4, n_estimators=3, eta=0.3, objective="squared"),
        "regularised": gbdt.GbdtParams(max_depth=5, n_estimators=6, eta=0.5, gamma=0.1, lam=2.0,
                                       min_child_weight=3.0),
    }
    data = {}
    for sname, (x, y) in sets.items():
        data[f"{sname}/x"] = np.asarray(x, np.float64)
        data[f"{sname}/y"] = np.asarray(y, np.int64)
        for pname, p in params.items():
            model = gbdt.fit_gbdt(x, y, p)
            data[f"{sname}/{pname}/model"] = np.array(gbdt.serialize_model(model))
            cv = gbdt.cross_validate(x, y, folds=5, params=p, seed=3)
            data[f"{sname}/{pname}/cv"] = np.array(json.dumps(
                [list(cv.fold_accuracies), list(cv.negative), list(cv.positive), list(cv.total)]))
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT} ({len(data)} arrays)")


if __name__ == "__main__":
    main()
