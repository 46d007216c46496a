"""B200-native MTNN hot path (arXiv 1702.03192): NT / TNN FP32 GEMMs + GBDT selector.

Drop-in for the reference package ``mtnn``'s hot-path API
(/root/reference/pkg/src/mtnn/__init__.py:10-76, the names below): the
kernels, the selector and the model format. Compute runs in the sm_100a
library ``lib/libmtnn_b200.so`` through its C-ABI (include/mtnn_b200.h);
there is no CPU fallback.
"""

from ._backend import active_backend
from .gbdt import (
    GbdtModel,
    GbdtParams,
    TreeNode,
    deserialize_model,
    load_model,
    predict,
    predict_raw,
    save_model,
    serialize_model,
)
from .kernels import ProblemShape, as_matrix, gemm_nn, gemm_nt, gemm_tnn, transpose_oop
from .platform import PlatformFeatures, probe_platform
from .selector import Dispatcher, SelectionDecision, build_features, mtnn_gemm, select

__version__ = "0.1.0"

__all__ = [
    "Dispatcher",
    "GbdtModel",
    "GbdtParams",
    "PlatformFeatures",
    "ProblemShape",
    "SelectionDecision",
    "TreeNode",
    "active_backend",
    "as_matrix",
    "build_features",
    "deserialize_model",
    "gemm_nn",
    "gemm_nt",
    "gemm_tnn",
    "load_model",
    "mtnn_gemm",
    "predict",
    "predict_raw",
    "probe_platform",
    "save_model",
    "select",
    "serialize_model",
    "transpose_oop",
]
