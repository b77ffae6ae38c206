"""Shared fixtures.  Markers: ``gpu`` = needs a B200 (run with -m gpu)."""

import json
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
MANIFEST = json.loads((GOLDEN / "manifest.json").read_text())


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def rel_err(a, b) -> float:
    """The reference suite's metric: max |a-b| / max(|b|, 1)
    (pkg/tests/conftest.py:85-93)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return np.inf
    if a.size == 0:
        return 0.0
    with np.errstate(invalid="ignore"):
        d = np.abs(a - b) / np.maximum(np.abs(b), 1.0)
    both_nan = np.isnan(a) & np.isnan(b)
    d = np.where(both_nan, 0.0, d)
    return float(np.max(np.nan_to_num(d, nan=np.inf)))


def load_case(case):
    d = np.load(GOLDEN / "vectors" / case["file"])
    inputs = {k[3:]: d[k] for k in d.files if k.startswith("in/")}
    return d, inputs


def golden_cases(max_per_kernel=None):
    out = []
    for name, ent in MANIFEST["kernels"].items():
        for v in ent["variants"]:
            cases = ent["cases"] if max_per_kernel is None else ent["cases"][:max_per_kernel]
            for case in cases:
                out.append((name, v, case))
    return out


@pytest.fixture(scope="session")
def manifest():
    return MANIFEST
