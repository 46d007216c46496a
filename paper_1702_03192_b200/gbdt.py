"""GBDT selector model: types, prediction and the JSON v1 wire format.

Mirrors the prediction/serialization half of the reference learner
(/root/reference/pkg/src/mtnn/gbdt.py): ``GbdtParams`` (:49-65), ``TreeNode``
(:68-95, routing ``x[f] < t`` -> left), ``GbdtModel`` (:98-103),
``predict_raw``/``predict``/``predict_batch`` (:242-269; label +1 = NT iff
raw >= 0), and ``serialize_model``/``deserialize_model`` (:388-455) with the
same document layout, so a model trained by the reference's ``fit_gbdt`` loads
here unchanged and vice versa. Training (exact-greedy CART boosting,
cross-validation) is host-side offline work and stays with the reference
learner; see DESIGN.md.

The hot-path evaluator is native: ``NativeModel`` packs the trees into the
C++ model handle of libmtnn_b200 (include/mtnn_b200.h ``mtnn_model_*``), whose
float64 walk is label-identical to ``predict`` on the same model.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = [
    "GbdtParams",
    "TreeNode",
    "GbdtModel",
    "NativeModel",
    "pack_trees",
    "predict",
    "predict_raw",
    "predict_batch",
    "accuracy",
    "serialize_model",
    "deserialize_model",
    "save_model",
    "load_model",
    "ModelFormatError",
]

MODEL_FORMAT_VERSION = 1


@dataclass(frozen=True)
class GbdtParams:
    max_depth: int = 8
    n_estimators: int = 8
    eta: float = 1.0
    gamma: float = 0.0
    lam: float = 1.0
    min_child_weight: float = 1.0
    objective: str = "logistic"

    def __post_init__(self):
        if self.max_depth < 1:
            raise ValueError(f"max_depth must be >= 1, got {self.max_depth}")
        if self.n_estimators < 1:
            raise ValueError(f"n_estimators must be >= 1, got {self.n_estimators}")
        if self.objective not in ("logistic", "squared"):
            raise ValueError(f"unknown objective {self.objective!r}")


@dataclass
class TreeNode:
    """Internal node (feature, threshold, children) or leaf (weight)."""

    feature: int | None = None
    threshold: float = 0.0
    left: "TreeNode | None" = None
    right: "TreeNode | None" = None
    weight: float = 0.0

    @property
    def is_leaf(self) -> bool:
        return self.feature is None

    def depth(self) -> int:
        if self.is_leaf:
            return 0
        return 1 + max(self.left.depth(), self.right.depth())

    def route(self, x) -> float:
        node = self
        while node.feature is not None:
            node = node.left if x[node.feature] < node.threshold else node.right
        return node.weight

    def node_count(self) -> int:
        if self.is_leaf:
            return 1
        return 1 + self.left.node_count() + self.right.node_count()


@dataclass(frozen=True)
class GbdtModel:
    trees: tuple
    params: GbdtParams
    base_score: float = 0.0
    n_features: int = 8


def predict_raw(model: GbdtModel, features) -> float:
    """Raw (log-odds) score: base_score + sum of eta-scaled leaf weights."""
    x = np.asarray(features, dtype=np.float64)
    if x.shape != (model.n_features,):
        raise ValueError(f"expected {model.n_features} features, got shape {x.shape}")
    if not np.isfinite(x).all():
        raise ValueError("features must be finite")
    raw = model.base_score
    eta = model.params.eta
    for tree in model.trees:
        raw += eta * tree.route(x)
    return raw


def predict(model: GbdtModel, features) -> int:
    """+1 (choose NT) when the raw score is >= 0, else -1 (choose TNN)."""
    return 1 if predict_raw(model, features) >= 0.0 else -1


def _tree_outputs(node: TreeNode, x: np.ndarray) -> np.ndarray:
    out = np.empty(x.shape[0], dtype=np.float64)
    stack = [(node, np.arange(x.shape[0]))]
    while stack:
        nd, idx = stack.pop()
        if nd.is_leaf:
            out[idx] = nd.weight
            continue
        go_left = x[idx, nd.feature] < nd.threshold
        stack.append((nd.left, idx[go_left]))
        stack.append((nd.right, idx[~go_left]))
    return out


def predict_batch(model: GbdtModel, x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2 or x.shape[1] != model.n_features:
        raise ValueError(f"expected an (n, {model.n_features}) array")
    raw = np.full(x.shape[0], model.base_score, dtype=np.float64)
    for tree in model.trees:
        raw += model.params.eta * _tree_outputs(tree, x)
    return np.where(raw >= 0.0, 1, -1)


def accuracy(model: GbdtModel, x, y) -> float:
    return float(np.mean(predict_batch(model, x) == np.asarray(y)))


# --------------------------------------------------------------------- packing
def pack_trees(model: GbdtModel):
    """Flatten trees into (feat, thresh, left, right, leaf) arrays.

    Same layout as the reference Dispatcher (selector.py:82-123): width = the
    largest node count, feat = -1 marks a leaf, nodes in pre-order with the
    root at 0, and an empty ensemble packs to one tree with a 0.0 leaf.
    """
    n_trees = max(len(model.trees), 1)
    width = max([t.node_count() for t in model.trees] or [1])
    feat = np.full((n_trees, width), -1, dtype=np.int64)
    thresh = np.zeros((n_trees, width), dtype=np.float64)
    left = np.zeros((n_trees, width), dtype=np.int64)
    right = np.zeros((n_trees, width), dtype=np.int64)
    leaf = np.zeros((n_trees, width), dtype=np.float64)
    for t, root in enumerate(model.trees):
        counter = [0]

        def emit(node):
            idx = counter[0]
            counter[0] += 1
            if node.is_leaf:
                leaf[t, idx] = node.weight
            else:
                feat[t, idx] = node.feature
                thresh[t, idx] = node.threshold
                left[t, idx] = emit(node.left)
                right[t, idx] = emit(node.right)
            return idx

        emit(root)
    return feat, thresh, left, right, leaf


class NativeModel:
    """Immutable C++ model handle (libmtnn_b200 ``mtnn_model``); thread-safe."""

    def __init__(self, handle: int, n_features: int):
        self._h = ctypes.c_void_p(handle)
        self.n_features = n_features

    @classmethod
    def from_model(cls, model: GbdtModel) -> "NativeModel":
        packed = pack_trees(model)
        feat, thresh, left, right, leaf = packed
        out = ctypes.c_void_p()
        _lib.check(_lib.lib.mtnn_model_from_packed(
            feat.ctypes.data_as(_lib._I64P), thresh.ctypes.data_as(_lib._DP),
            left.ctypes.data_as(_lib._I64P), right.ctypes.data_as(_lib._I64P),
            leaf.ctypes.data_as(_lib._DP), feat.shape[0], feat.shape[1],
            float(model.base_score), float(model.params.eta), int(model.n_features),
            ctypes.byref(out)))
        return cls(out.value, int(model.n_features))

    @classmethod
    def from_json(cls, text: str | bytes) -> "NativeModel":
        data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
        out = ctypes.c_void_p()
        rc = _lib.lib.mtnn_model_load_json(data, len(data), ctypes.byref(out))
        if rc != _lib.OK:
            raise ModelFormatError(_lib.last_error())
        return cls(out.value, int(_lib.lib.mtnn_model_n_features(out)))

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def raw(self, features) -> float:
        x = np.ascontiguousarray(features, dtype=np.float64).reshape(-1)
        r = ctypes.c_double()
        _lib.check(_lib.lib.mtnn_model_raw(self._h, x.ctypes.data_as(_lib._DP), x.size,
                                           ctypes.byref(r)))
        return r.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is None or not h.value:
            return
        try:
            _lib.lib.mtnn_model_free(h)
        except AttributeError:  # interpreter shutdown: module globals already cleared
            pass
        self._h = ctypes.c_void_p()


# --------------------------------------------------------------- serialization
class ModelFormatError(ValueError):
    """Malformed model document; the message carries the JSON location."""


def _node_doc(node: TreeNode):
    if node.is_leaf:
        return {"leaf": node.weight}
    return {"feat": node.feature, "thresh": node.threshold,
            "left": _node_doc(node.left), "right": _node_doc(node.right)}


def serialize_model(model: GbdtModel) -> str:
    """JSON v1 document; floats keep round-trip (repr) precision."""
    p = model.params
    doc = {
        "version": MODEL_FORMAT_VERSION,
        "params": {"max_depth": p.max_depth, "n_estimators": p.n_estimators, "eta": p.eta,
                   "gamma": p.gamma, "lambda": p.lam, "min_child_weight": p.min_child_weight,
                   "objective": p.objective},
        "base_score": model.base_score,
        "n_features": model.n_features,
        "trees": [_node_doc(t) for t in model.trees],
    }
    return json.dumps(doc, indent=1)


def _node_from_doc(obj, where: str) -> TreeNode:
    if not isinstance(obj, dict):
        raise ModelFormatError(f"{where}: expected an object, got {type(obj).__name__}")
    if "leaf" in obj:
        if not isinstance(obj["leaf"], (int, float)):
            raise ModelFormatError(f"{where}.leaf: expected a number")
        return TreeNode(weight=float(obj["leaf"]))
    for key in ("feat", "thresh", "left", "right"):
        if key not in obj:
            raise ModelFormatError(f"{where}: missing {key!r}")
    feat = obj["feat"]
    if not isinstance(feat, int) or feat < 0:
        raise ModelFormatError(f"{where}.feat: expected a non-negative integer")
    return TreeNode(feature=feat, threshold=float(obj["thresh"]),
                    left=_node_from_doc(obj["left"], where + ".left"),
                    right=_node_from_doc(obj["right"], where + ".right"))


def deserialize_model(text: str | bytes) -> GbdtModel:
    if isinstance(text, bytes):
        text = text.decode("utf-8")
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ModelFormatError(
            f"not valid JSON at line {exc.lineno} column {exc.colno}: {exc.msg}") from exc
    if not isinstance(doc, dict):
        raise ModelFormatError("$: expected a JSON object")
    for key in ("version", "params", "base_score", "trees"):
        if key not in doc:
            raise ModelFormatError(f"$: missing {key!r}")
    if doc["version"] != MODEL_FORMAT_VERSION:
        raise ModelFormatError(f"$.version: unsupported version {doc['version']!r}")
    rp = doc["params"]
    if not isinstance(rp, dict):
        raise ModelFormatError("$.params: expected an object")
    try:
        params = GbdtParams(
            max_depth=int(rp["max_depth"]), n_estimators=int(rp["n_estimators"]),
            eta=float(rp["eta"]), gamma=float(rp["gamma"]), lam=float(rp["lambda"]),
            min_child_weight=float(rp["min_child_weight"]),
            objective=str(rp.get("objective", "logistic")))
    except KeyError as exc:
        raise ModelFormatError(f"$.params: missing {exc.args[0]!r}") from None
    except (TypeError, ValueError) as exc:
        raise ModelFormatError(f"$.params: {exc}") from None
    if not isinstance(doc["trees"], list):
        raise ModelFormatError("$.trees: expected a list")
    trees = tuple(_node_from_doc(o, f"$.trees[{i}]") for i, o in enumerate(doc["trees"]))
    if len(trees) > params.n_estimators:
        raise ModelFormatError(
            f"$.trees: {len(trees)} trees exceeds n_estimators={params.n_estimators}")
    return GbdtModel(trees=trees, params=params, base_score=float(doc["base_score"]),
                     n_features=int(doc.get("n_features", 8)))


def save_model(model: GbdtModel, path) -> None:
    with open(path, "w") as fh:
        fh.write(serialize_model(model))


def load_model(path) -> GbdtModel:
    with open(path) as fh:
        return deserialize_model(fh.read())
