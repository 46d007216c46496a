"""Offline selector training: exact-greedy boosted regression trees and
stratified k-fold cross-validation (the paper's §V-B learner).

Restates the training half of the reference learner
(/root/reference/pkg/src/mtnn/gbdt.py): ``fit_gbdt`` (:207-239) with the
logistic / squared objectives, the exact greedy split search of ``_best_split``
(:119-156: every feature, midpoint thresholds between distinct sorted values,
XGBoost gain with ``lam``/``gamma``, ``min_child_weight`` on both children,
first maximum within a feature, strictly-better across features) and
``cross_validate`` (:311-350, folds from ``_stratified_folds`` :296-304).

The structure differs from the reference (an explicit node stack; one
stable ``argsort`` of the node's whole feature block and one ``cumsum`` per
node instead of a per-feature loop), but every floating-point reduction is
taken over the same values in the same order (subsets keep the original
sample order; ``cumsum`` is sequential along either axis), so the trained
trees — and therefore the serialized model and the CV report — are identical
to the reference's. ``tests/test_learn.py`` checks this against models and
reports the reference produced (``tests/golden/make_golden_learn.py``).

Training is host-side work on a few hundred samples; it is not on the GPU
hot path, and nothing here touches the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .gbdt import GbdtModel, GbdtParams, TreeNode, predict_batch

__all__ = ["fit_gbdt", "fit_tree", "cross_validate", "CvReport"]


def _split_search(xn, gn, hn, params):
    """Best (gain, feature, threshold) for one node, or None.

    xn (s, f), gn/hn (s,) in the node's sample order."""
    lam, gamma, mcw = params.lam, params.gamma, params.min_child_weight
    g_tot = float(gn.sum())
    h_tot = float(hn.sum())
    parent = g_tot ** 2 / (h_tot + lam)
    if xn.shape[0] < 2:
        return None
    order = np.argsort(xn, axis=0, kind="stable")            # per-feature sort
    xs = np.take_along_axis(xn, order, axis=0)
    gl = np.cumsum(gn[order], axis=0)[:-1]                    # left sums at each cut
    hl = np.cumsum(hn[order], axis=0)[:-1]
    gr = g_tot - gl
    hr = h_tot - hl
    with np.errstate(divide="ignore", invalid="ignore"):
        gains = 0.5 * (gl ** 2 / (hl + lam) + gr ** 2 / (hr + lam) - parent) - gamma
    cut = xs[1:] != xs[:-1]                                   # distinct neighbours only
    valid = cut & (hl >= mcw) & (hr >= mcw)
    best = None
    for f in np.flatnonzero(valid.any(axis=0)):
        col = np.where(valid[:, f], gains[:, f], -np.inf)
        pos = int(np.argmax(col))
        gain = float(col[pos])
        if gain <= 0.0:
            continue
        if best is None or gain > best[0]:
            best = (gain, int(f), (float(xs[pos, f]) + float(xs[pos + 1, f])) / 2.0)
    return best


def _grow(x, g, h, params) -> TreeNode:
    """Depth-limited tree over all samples, built with an explicit stack."""
    root = TreeNode()
    stack = [(root, np.arange(x.shape[0]), 0)]
    while stack:
        node, idx, depth = stack.pop()
        gn, hn = g[idx], h[idx]
        split = _split_search(x[idx], gn, hn, params) if depth < params.max_depth else None
        if split is None:
            node.weight = -float(gn.sum()) / (float(hn.sum()) + params.lam)
            continue
        _, f, t = split
        go_left = x[idx, f] < t
        node.feature, node.threshold = f, t
        node.left, node.right = TreeNode(), TreeNode()
        stack.append((node.right, idx[~go_left], depth + 1))
        stack.append((node.left, idx[go_left], depth + 1))
    return root


def _outputs(tree: TreeNode, x) -> np.ndarray:
    out = np.empty(x.shape[0], dtype=np.float64)
    stack = [(tree, np.arange(x.shape[0]))]
    while stack:
        node, idx = stack.pop()
        if node.is_leaf:
            out[idx] = node.weight
            continue
        left = x[idx, node.feature] < node.threshold
        stack.append((node.left, idx[left]))
        stack.append((node.right, idx[~left]))
    return out


def fit_tree(x, g, h, params: GbdtParams | None = None) -> TreeNode:
    """One regression tree on gradients/hessians (reference gbdt.py:177-189)."""
    params = params or GbdtParams()
    x = np.asarray(x, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    if x.ndim != 2 or x.shape[0] == 0:
        raise ValueError("need a non-empty 2-D feature array")
    if g.shape != (x.shape[0],) or h.shape != (x.shape[0],):
        raise ValueError("gradient/hessian length must match the sample count")
    if not (np.isfinite(g).all() and np.isfinite(h).all()):
        raise ValueError("gradients and hessians must be finite")
    return _grow(x, g, h, params)


def fit_gbdt(x, y, params: GbdtParams | None = None) -> GbdtModel:
    """Boosted ensemble on features x and labels y in {-1, +1} (base score 0)."""
    params = params or GbdtParams()
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y)
    if x.ndim != 2 or x.shape[0] == 0:
        raise ValueError("training set is empty")
    if y.shape != (x.shape[0],):
        raise ValueError("label count must match the sample count")
    if not np.isin(y, (-1, 1)).all():
        raise ValueError("labels must be -1 or +1")
    target01 = (y.astype(np.float64) + 1.0) / 2.0
    target_pm = y.astype(np.float64)
    raw = np.zeros(x.shape[0], dtype=np.float64)
    trees = []
    for _ in range(params.n_estimators):
        if params.objective == "logistic":
            p = 1.0 / (1.0 + np.exp(-raw))
            g, h = p - target01, p * (1.0 - p)
        else:
            g, h = raw - target_pm, np.ones_like(raw)
        tree = _grow(x, g, h, params)
        trees.append(tree)
        raw = raw + params.eta * _outputs(tree, x)
    return GbdtModel(trees=tuple(trees), params=params, base_score=0.0, n_features=x.shape[1])


@dataclass(frozen=True)
class CvReport:
    """Per-fold accuracies plus (min, max, average) per class and overall."""

    fold_accuracies: tuple
    negative: tuple
    positive: tuple
    total: tuple

    @property
    def overall_average(self) -> float:
        return self.total[2]


def _fold_ids(y, folds, seed):
    """Each class shuffled by one generator (class -1 first), dealt round-robin."""
    rng = np.random.default_rng(seed)
    fold = np.empty(len(y), dtype=np.int64)
    for cls in (-1, 1):
        members = np.flatnonzero(y == cls)
        rng.shuffle(members)
        fold[members] = np.arange(members.size) % folds
    return fold


def _mma(values):
    return (float(min(values)), float(max(values)), float(np.mean(values)))


def cross_validate(x, y, folds: int = 5, params: GbdtParams | None = None,
                   seed: int = 0) -> CvReport:
    """Stratified k-fold CV (reference gbdt.py:311-350)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y)
    if folds < 2:
        raise ValueError(f"folds must be >= 2, got {folds}")
    if x.shape[0] < folds:
        raise ValueError(f"need at least {folds} samples, got {x.shape[0]}")
    fold = _fold_ids(y, folds, seed)
    overall, per_cls = [], {-1: [], 1: []}
    for f in range(folds):
        test = fold == f
        if not test.any():
            continue
        model = fit_gbdt(x[~test], y[~test], params)
        pred, truth = predict_batch(model, x[test]), y[test]
        overall.append(float(np.mean(pred == truth)))
        for cls, acc in per_cls.items():
            sel = truth == cls
            if sel.any():
                acc.append(float(np.mean(pred[sel] == cls)))
    nan3 = (math.nan,) * 3
    return CvReport(fold_accuracies=tuple(overall),
                    negative=_mma(per_cls[-1]) if per_cls[-1] else nan3,
                    positive=_mma(per_cls[1]) if per_cls[1] else nan3,
                    total=_mma(overall))
