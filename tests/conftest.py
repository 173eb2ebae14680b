"""Shared test setup.

Markers: `gpu` tests need a B200 (run on the GPU box with `-m gpu`); all
others run on CPU.  The oracle (oracle/) is the checker: tests import it,
the product package never does.
"""
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_models():
    return json.loads((GOLDEN / "models.json").read_text())


def model_path(name: str) -> Path:
    return GOLDEN / golden_models()[name]["path"]


@pytest.fixture(scope="session")
def models():
    return golden_models()


@pytest.fixture(scope="session")
def fig_path():
    return GOLDEN / "models" / "fig1" / "net.exp"
