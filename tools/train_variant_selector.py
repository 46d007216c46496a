"""Can the MTNN learner pick the B200 tensor-core *variants* better than the
hand rules? (on the B200 the NT/TNN decision is trivial —
NT wins ~507/512 — while the variant choices inside tc3xf16s are thresholds.)

    python tools/train_variant_selector.py profiles/variants_r02.csv

Input: per-shape interleaved timings of two decisions over the configs[1] sweep
(tools/probes/probe_variant_sweep.py): `pair` (single-CTA 128x256 tiles vs CTA
pairs 256x256) and `ink` (pre-split operands vs the long operand split inside
the GEMM). For each decision: labels (+1 iff variant 1 is faster), the
reference learner (paper_1702_03192_b200.learn: fit_gbdt / cross_validate,
default parameters, features = the selector's platform vector + (m, n, k)),
and the sweep time under the hand rule, the learned choice (out-of-fold: each
case predicted by the model trained without its fold) and the per-shape
oracle. Writes profiles/variant_selector_r02.json."""
import csv
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1702_03192_b200 import gbdt, learn  # noqa: E402

RULES = {
    "pair": lambda m, n, k: ((m + 255) // 256) * ((n + 255) // 256) >= 74,
    "ink": lambda m, n, k: min(m, n) <= 256 and max(m, n) >= 1024,
}


def main(path, out=ROOT / "profiles" / "variant_selector_r02.json"):
    rows = list(csv.DictReader(open(path)))
    platform = json.loads((ROOT / "paper_1702_03192_b200" / "models" / "b200_sweep.report.json")
                          .read_text())["platform"]
    report = {"source": str(path), "platform": platform}
    for name, rule in RULES.items():
        rs = [r for r in rows if r["decision"] == name]
        mnk = np.array([(int(r["m"]), int(r["n"]), int(r["k"])) for r in rs])
        t0 = np.array([float(r["t0"]) for r in rs])
        t1 = np.array([float(r["t1"]) for r in rs])
        x = np.array([tuple(platform) + tuple(float(v) for v in row) for row in mnk])
        y = np.where(t1 < t0, 1, -1)
        cv = learn.cross_validate(x, y, folds=5, seed=0)
        # out-of-fold choices: the same stratified folds as cross_validate
        fold = learn._fold_ids(y, 5, 0)
        pick = np.zeros(len(y), int)
        for f in range(5):
            te = fold == f
            model = learn.fit_gbdt(x[~te], y[~te])
            pick[te] = gbdt.predict_batch(model, x[te])
        t_rule = float(np.where([rule(*v) for v in mnk], t1, t0).sum())
        t_learn = float(np.where(pick == 1, t1, t0).sum())
        t_best = float(np.minimum(t0, t1).sum())
        report[name] = {
            "cases": len(rs), "variant1_wins": int((y == 1).sum()),
            "cv_5fold_total(min,max,avg)": cv.total,
            "rule_label_accuracy": float(np.mean([rule(*v) == (l == 1) for v, l in zip(mnk, y)])),
            "sweep_ms": {"variant0": float(t0.sum() * 1e3), "variant1": float(t1.sum() * 1e3),
                         "hand_rule": t_rule * 1e3, "learned_out_of_fold": t_learn * 1e3,
                         "per_shape_best": t_best * 1e3},
        }
    Path(out).write_text(json.dumps(report, indent=1))
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
