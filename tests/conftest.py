"""Shared fixtures.  Markers: ``gpu`` (needs a B200 + the built CUDA library)."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

import paper_2009_02823_b200 as sv  # noqa: E402
from cases import input_state  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and libsvgb200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name: str = "golden_small.json") -> dict:
    path = os.path.join(HERE, "golden", name)
    if not os.path.exists(path):
        pytest.skip(f"fixture {name} not generated")
    with open(path) as f:
        return json.load(f)["cases"]


def cvec(pairs) -> np.ndarray:
    a = np.asarray(pairs, dtype=float).reshape(-1, 2)
    return a[:, 0] + 1j * a[:, 1]


def materialize(build):
    """Build a case with THIS package's API: (circuit, theta, obs, input_state, method)."""
    spec = build(sv)
    circ = spec["circuit"]
    return circ, spec["theta"], spec["obs"], input_state(sv, circ.num_qubits, spec["input"]), spec["method"]


def close(actual, expected, tol) -> bool:
    """abs-or-rel: |a-e| <= tol * max(1, |e|) elementwise."""
    actual, expected = np.asarray(actual), np.asarray(expected)
    return bool(np.all(np.abs(actual - expected) <= tol * np.maximum(1.0, np.abs(expected))))


def max_err(actual, expected) -> float:
    actual, expected = np.asarray(actual), np.asarray(expected)
    if actual.size == 0:
        return 0.0
    return float(np.max(np.abs(actual - expected) / np.maximum(1.0, np.abs(expected))))


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
