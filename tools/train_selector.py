"""Retrain the MTNN selector on B200-measured sweep timings.

    python tools/train_selector.py gpurun_out/sweep_auto.csv

Pipeline (the reference's §V-B recipe, all in-package): the timings CSV
(sweep.read_timings_csv; wire format of the reference bench.py:341-363) ->
labels (+1 iff p_nt - p_tnn >= 0, sweep.label_of = bench.py:296-303) ->
5-fold stratified cross_validate + fit_gbdt with default GbdtParams (8 trees,
depth 8, eta 1, gamma 0) from paper_1702_03192_b200.learn (model-identical to
the reference learner, tests/test_learn.py) -> serialize_model. Writes
paper_1702_03192_b200/models/b200_sweep.json and a report next to it.
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1702_03192_b200 import gbdt, learn, sweep  # noqa: E402


def samples(timings: dict, platform):
    rows = sorted(sweep.rows_from_timings(timings), key=lambda r: (r.m, r.n, r.k))
    x = np.array([tuple(platform) + (float(r.m), float(r.n), float(r.k)) for r in rows])
    y = np.array([sweep.label_of(r) for r in rows])
    return rows, x, y


def main(csv_path, out_name="b200_sweep"):
    meta = json.loads(Path(csv_path + ".platform.json").read_text())
    rows, x, y = samples(sweep.read_timings_csv(csv_path), meta["platform"])
    cv = learn.cross_validate(x, y, folds=5, seed=0)
    model = learn.fit_gbdt(x, y)
    out = ROOT / "paper_1702_03192_b200" / "models"
    out.mkdir(exist_ok=True)
    (out / f"{out_name}.json").write_text(gbdt.serialize_model(model))
    ratio = np.array([r.t_nt / r.t_tnn for r in rows])  # p_tnn / p_nt
    report = {
        "source": os.path.basename(csv_path), "platform": meta["platform"],
        "cases": len(rows), "labels": {"+1 (NT)": int((y == 1).sum()), "-1 (TNN)": int((y == -1).sum())},
        "cv_5fold": {"fold_accuracies": cv.fold_accuracies, "negative(min,max,avg)": cv.negative,
                     "positive(min,max,avg)": cv.positive, "total(min,max,avg)": cv.total},
        "train_accuracy": gbdt.accuracy(model, x, y),
        "mean_p_tnn_over_p_nt": float(np.mean(ratio)),
        "learner": "paper_1702_03192_b200.learn.fit_gbdt, default GbdtParams (8 trees, depth 8, "
                   "eta 1, gamma 0)",
    }
    (out / f"{out_name}.report.json").write_text(json.dumps(report, indent=1))
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
