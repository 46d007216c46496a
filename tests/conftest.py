"""Shared fixtures. Tests needing a B200 carry @pytest.mark.gpu; everything else
runs on CPU (the C-ABI library loads without a GPU; the oracle is plain C)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))

# The two reference platform rows used throughout the reference tests
# (/root/reference/pkg/tests/conftest.py:12-13).
PLATFORM_A = {"gm": 8, "sm": 20, "cc": 1607, "mbw": 256, "l2c": 2048}
PLATFORM_B = {"gm": 10, "sm": 28, "cc": 1417, "mbw": 384, "l2c": 3072}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run with -m gpu)")


@pytest.fixture
def platform_a():
    from paper_1702_03192_b200.platform import PlatformFeatures

    return PlatformFeatures(**{k: float(v) for k, v in PLATFORM_A.items()})


@pytest.fixture
def rng() -> np.random.Generator:
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def golden_kernels():
    return dict(np.load(GOLDEN / "kernels.npz"))


@pytest.fixture(scope="session")
def golden_selector():
    return dict(np.load(GOLDEN / "selector.npz"))


@pytest.fixture(scope="session")
def golden_operands():
    return dict(np.load(GOLDEN / "operands.npz"))


def golden_model_names():
    return sorted(p.stem for p in (GOLDEN / "models").glob("*.json"))


def golden_model_text(name: str) -> str:
    return (GOLDEN / "models" / f"{name}.json").read_text()
