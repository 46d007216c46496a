"""The paper's evaluation (Table V: MTNN vs NT / TNN, GOW avg/max, LUB avg/min,
the p_mtnn/p_nt histogram) on the B200, with the reference acceptance test's
held-out protocol (pkg/tests/test_acceptance.py:166-188).

    python tools/eval_report.py [--exp-min 7] [--exp-max 14] [--out profiles/eval_r02]

1. sweep: NN / NT / TNN timed per case (CUDA events, interleaved, L2 flushed,
   median of --reps), written in the reference's timings CSV format;
2. labels (+1 iff p_nt >= p_tnn) and the full-data model (learn.fit_gbdt,
   default GbdtParams) plus its 5-fold stratified CV report;
3. held-out: split_holdout(shapes, 0.2, seed 7) like the acceptance test, a
   model trained on the other 80 %, evaluate_cases(remeasured) on the held-out
   shapes -> aggregate; TNN-class recall on those shapes;
4. the full-data model evaluated on all shapes (remeasured), as the paper's
   Table V does (its model saw every case).
Outputs <out>.json and <out>.md (+ the timings CSV).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1702_03192_b200 import evaluate, gbdt, learn, sweep  # noqa: E402
from paper_1702_03192_b200.cli import split_holdout  # noqa: E402
from paper_1702_03192_b200.kernels import ProblemShape  # noqa: E402
from paper_1702_03192_b200.platform import probe_platform  # noqa: E402
from paper_1702_03192_b200.selector import Dispatcher  # noqa: E402

PAPER_TOTAL = {"mtnn_vs_nt": 54.03, "mtnn_vs_tnn": 21.92, "gow_avg": 76.23, "gow_max": 1439.39,
               "lub_avg": -0.28, "lub_min": -71.62}  # PAPER.md:388-396 (GTX1080 + TitanX)


def report_dict(rep):
    return {"mtnn_vs_nt": rep.mtnn_vs_nt, "mtnn_vs_tnn": rep.mtnn_vs_tnn, "gow_avg": rep.gow_avg,
            "gow_max": rep.gow_max, "lub_avg": rep.lub_avg, "lub_min": rep.lub_min,
            "n_cases": rep.n_cases, "p_mtnn_mode": rep.p_mtnn_mode,
            "histogram_p_mtnn_over_p_nt": list(rep.ratio_histogram)}


def recall(cases):
    tnn_faster = [c for c in cases if c.p_tnn > c.p_nt]
    picked = [c for c in tnn_faster if c.decision is not None and c.decision.choice.value == "tnn"]
    nt_faster = [c for c in cases if c.p_tnn <= c.p_nt]
    nt_ok = [c for c in nt_faster if c.decision is not None and c.decision.choice.value == "nt"]
    return {"tnn_faster_cases": len(tnn_faster), "tnn_recall": (len(picked) / len(tnn_faster)
                                                                 if tnn_faster else None),
            "nt_faster_cases": len(nt_faster), "nt_recall": (len(nt_ok) / len(nt_faster)
                                                              if nt_faster else None)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--exp-min", type=int, default=7)
    ap.add_argument("--exp-max", type=int, default=14)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--eval-reps", type=int, default=9)  # EVAL_CONFIG reps (test_acceptance.py:28)
    ap.add_argument("--out", default="gpurun_out/eval_r02")
    args = ap.parse_args()
    t0 = time.time()
    plat = probe_platform()
    exps = range(args.exp_min, args.exp_max + 1)
    rows = sweep.sweep(exps, reps=args.reps, warmup=2)
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    sweep.write_timings_csv(str(out) + ".csv", rows)
    x = np.array([tuple(plat.as_tuple()) + (float(r.m), float(r.n), float(r.k)) for r in rows])
    y = np.array([sweep.label_of(r) for r in rows])
    shapes = [ProblemShape(r.m, r.n, r.k) for r in rows]
    full = learn.fit_gbdt(x, y)
    cv = learn.cross_validate(x, y, folds=5, seed=0)
    # held-out protocol (test_acceptance.py:166-188)
    _, held = split_holdout([tuple(s) for s in shapes], 0.2, 7)
    held_keys = {tuple(s) for s in held}
    keep = np.array([tuple(s) not in held_keys for s in shapes])
    model_80 = learn.fit_gbdt(x[keep], y[keep])
    held_shapes = [ProblemShape(*s) for s in held]
    held_cases = evaluate.evaluate_cases(Dispatcher(model_80, plat), held_shapes,
                                         reps=args.eval_reps, warmup=2, p_mtnn_mode="remeasured")
    held_rep = evaluate.aggregate(held_cases, "remeasured")
    all_cases = evaluate.evaluate_cases(Dispatcher(full, plat), shapes, reps=args.eval_reps,
                                        warmup=2, p_mtnn_mode="remeasured")
    all_rep = evaluate.aggregate(all_cases, "remeasured")
    res = {
        "platform": plat.as_tuple(), "cases": len(rows),
        "labels": {"nt": int((y == 1).sum()), "tnn": int((y == -1).sum())},
        "cv_5fold": {"total(min,max,avg)": cv.total, "negative_tnn(min,max,avg)": cv.negative,
                     "positive_nt(min,max,avg)": cv.positive},
        "train_accuracy_full": gbdt.accuracy(full, x, y),
        "held_out": {"protocol": "split_holdout(shapes, 0.2, seed 7); model trained on the other "
                                 "80%; evaluate_cases remeasured (Dispatcher.gemm timed)",
                     **report_dict(held_rep), **recall(held_cases)},
        "all_cases_full_model": {**report_dict(all_rep), **recall(all_cases)},
        "paper_table_v_total": PAPER_TOTAL,
        "mean_p_tnn_over_p_nt": float(np.mean([r.t_nt / r.t_tnn for r in rows])),
        "seconds": time.time() - t0,
    }
    Path(str(out) + ".json").write_text(json.dumps(res, indent=1))
    lines = ["| Metric (%) | B200 held-out (20 %) | B200 all cases | paper (GTX1080+TitanX) |",
             "|---|---|---|---|"]
    for key, name in (("mtnn_vs_nt", "MTNN vs NT"), ("mtnn_vs_tnn", "MTNN vs TNN"),
                      ("gow_avg", "GOW avg"), ("gow_max", "GOW max"), ("lub_avg", "LUB avg"),
                      ("lub_min", "LUB min")):
        lines.append(f"| {name} | {res['held_out'][key]:.2f} | "
                     f"{res['all_cases_full_model'][key]:.2f} | {PAPER_TOTAL[key]:.2f} |")
    lines += ["", f"labels: NT faster {res['labels']['nt']}, TNN faster {res['labels']['tnn']}; "
              f"5-fold CV total avg {cv.total[2]:.3f}, TNN class avg {cv.negative[2]}; "
              f"held-out TNN recall {res['held_out']['tnn_recall']} "
              f"({res['held_out']['tnn_faster_cases']} TNN-faster cases)"]
    Path(str(out) + ".md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
