"""Retrain the MTNN selector on B200-measured sweep timings with the REFERENCE
learner, unchanged (build container only: imports /root/reference).

    python tools/train_selector.py gpurun_out/sweep_auto.csv

Pipeline = the reference's own fixture mode: read_timings_csv (bench.py:353-363)
-> sweep_grid(injected=...) (bench.py:243-293) -> label_records (+1 iff
p_nt - p_tnn >= 0, bench.py:296-309) -> cross_validate (gbdt.py:311-345, 5-fold
stratified) + fit_gbdt (gbdt.py:207-239, 8 trees depth 8 eta 1 gamma 0) ->
serialize_model. Writes paper_1702_03192_b200/models/b200_sweep.json and a
report next to it.
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb_train")

from mtnn import bench, gbdt  # noqa: E402  (the reference)
from mtnn.platform import PlatformFeatures  # noqa: E402


def main(csv_path):
    meta = json.loads(Path(csv_path + ".platform.json").read_text())
    plat = PlatformFeatures(*meta["platform"])
    timings = bench.read_timings_csv(csv_path)
    exps = sorted({int(np.log2(m)) for (m, _, _) in timings})
    records = bench.sweep_grid(range(exps[0], exps[-1] + 1), plat, injected=timings)
    samples = bench.label_records(records, plat)
    x, y = bench.samples_to_arrays(samples)
    cv = gbdt.cross_validate(x, y, folds=5, seed=0)
    model = gbdt.fit_gbdt(x, y)
    train_acc = gbdt.accuracy(model, x, y)
    out = ROOT / "paper_1702_03192_b200" / "models"
    out.mkdir(exist_ok=True)
    (out / "b200_sweep.json").write_text(gbdt.serialize_model(model))
    p_nt = np.array([r.p_nt for r in records]); p_tnn = np.array([r.p_tnn for r in records])
    report = {
        "source": os.path.basename(csv_path), "platform": meta["platform"],
        "cases": len(records), "labels": {"+1 (NT)": int((y == 1).sum()), "-1 (TNN)": int((y == -1).sum())},
        "cv_5fold": {"fold_accuracies": cv.fold_accuracies, "negative(min,max,avg)": cv.negative,
                     "positive(min,max,avg)": cv.positive, "total(min,max,avg)": cv.total},
        "train_accuracy": train_acc,
        "mean_p_tnn_over_p_nt": float(np.mean(p_tnn / p_nt)),
        "learner": "reference mtnn.gbdt.fit_gbdt, default GbdtParams (8 trees, depth 8, eta 1, gamma 0)",
    }
    (out / "b200_sweep.report.json").write_text(json.dumps(report, indent=1))
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
