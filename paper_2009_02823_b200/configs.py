"""Pinned BASELINE.json workloads (cfg 1-5) as circuit/observable builders.

BASELINE.json leaves layer order, seeds and random-term recipes open; they are
pinned here once and every test, fixture and
bench line goes through these functions.

The builders take an ``api`` namespace with the factory names the reference
exports at its package root (``Circuit``, ``Observable``, ``rx``, ``ry``,
``rz``, ``cx``, ``cry``, ``rp`` -- reference ``svgrad/__init__.py:3-53``), so
the SAME code builds the reference objects (golden-fixture generation, in this
container only) and this package's objects (tests, bench).

Seeds: H draws from ``np.random.default_rng([seed, cfg, 1])``, theta from
``np.random.default_rng([seed, cfg, 2]).uniform(0, 2*pi, P)``, seed = 0.
Random Pauli term: weight w ~ U{1..4}, qubits ``rng.choice(n, w, replace=False)``,
letters ~ U{X,Y,Z}, coefficient ~ N(0, 1), drawn in that order per term.
"""
from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np

NUM_CONFIGS = 5
DEFAULT_QUBITS = {1: 10, 2: 20, 3: 26, 4: 30, 5: 33}
_LETTERS = "XYZ"


def _default_api():
    from . import ir, operators

    return SimpleNamespace(
        Circuit=ir.Circuit, Observable=operators.Observable, rx=ir.rx, ry=ir.ry,
        rz=ir.rz, cx=ir.cx, cry=ir.cry, rp=ir.rp,
    )


@dataclass(frozen=True)
class Workload:
    cfg: int
    num_qubits: int
    circuit: object
    observable: object
    theta: np.ndarray

    @property
    def num_gates(self) -> int:
        return len(self.circuit.gates)

    @property
    def state_bytes(self) -> int:
        return 16 << self.num_qubits


def _rot(api, axis: str, q: int, p: int):
    return {"X": api.rx, "Y": api.ry, "Z": api.rz}[axis](q, p)


def _circuit(api, cfg: int, n: int):
    gates = []
    p = 0

    def take() -> int:
        nonlocal p
        p += 1
        return p - 1

    if cfg == 1:
        for _ in range(4):
            for axis in "XYZ":
                gates += [_rot(api, axis, q, take()) for q in range(n)]
            gates += [api.cx(i, i + 1) for i in range(n - 1)]
    elif cfg == 2:
        for _ in range(10):
            for axis in "YZ":
                gates += [_rot(api, axis, q, take()) for q in range(n)]
            gates += [api.cx(i, (i + 1) % n) for i in range(n)]
    elif cfg == 3:
        pairs = (("X", "Y"), ("Y", "Z"), ("Z", "X"))
        for layer in range(20):
            for axis in pairs[layer % 3]:
                gates += [_rot(api, axis, q, take()) for q in range(n)]
            gates += [api.cry(i, i + 1, take()) for i in range(n - 1)]
            gates += [api.rp("ZZ", (i, i + 1), take()) for i in range(n - 1)]
    elif cfg == 4:
        for _ in range(16):
            for axis in "YZ":
                gates += [_rot(api, axis, q, take()) for q in range(n)]
            gates += [api.cx(i, i + 1) for i in range(n - 1)]
    elif cfg == 5:
        for _ in range(12):
            for axis in "XYZ":
                gates += [_rot(api, axis, q, take()) for q in range(n)]
            gates += [api.rp("ZZ", (i, i + 1), take()) for i in range(n - 1)]
    else:
        raise ValueError(f"unknown config {cfg}")
    return api.Circuit(n, tuple(gates), p)


def _letters(n: int, placed: dict[int, str]) -> str:
    return "".join(placed.get(q, "I") for q in range(n))


def random_pauli_terms(n: int, count: int, rng: np.random.Generator):
    terms = []
    for _ in range(count):
        w = int(rng.integers(1, 5))
        qubits = rng.choice(n, size=min(w, n), replace=False)
        letters = rng.integers(0, 3, size=len(qubits))
        coeff = float(rng.normal())
        terms.append((coeff, _letters(n, {int(q): _LETTERS[int(l)] for q, l in zip(qubits, letters)})))
    return terms


def _observable(api, cfg: int, n: int, seed: int):
    rng = np.random.default_rng([seed, cfg, 1])
    if cfg in (1, 4):
        h = 1.0 if cfg == 1 else 0.7
        terms = [(1.0, _letters(n, {i: "Z", i + 1: "Z"})) for i in range(n - 1)]
        terms += [(h, _letters(n, {i: "X"})) for i in range(n)]
    elif cfg == 2:
        terms = random_pauli_terms(n, 64, rng)
    elif cfg == 3:
        terms = [
            (1.0, _letters(n, {i: a, i + 1: a})) for i in range(n - 1) for a in "XYZ"
        ]
    elif cfg == 5:
        terms = random_pauli_terms(n, 128, rng)
    else:
        raise ValueError(f"unknown config {cfg}")
    return api.Observable(n, tuple(terms))


def shard_flip_terms(observable, shard_qubits) -> int:
    """Number of terms with an X or Y factor on any of ``shard_qubits``."""
    return sum(
        any(factors[q] in "XY" for q in shard_qubits) for _, factors in observable.terms
    )


def build_workload(cfg: int, num_qubits: int | None = None, seed: int = 0, api=None) -> Workload:
    """Circuit, observable and theta of BASELINE.json ``configs[cfg-1]``.

    ``num_qubits`` rescales the same layer structure (reduced-size parity
    cases); the default is the configured size.
    """
    if cfg not in DEFAULT_QUBITS:
        raise ValueError(f"unknown config {cfg}")
    api = api or _default_api()
    n = DEFAULT_QUBITS[cfg] if num_qubits is None else int(num_qubits)
    if n < 2:
        raise ValueError("workloads need at least two qubits")
    circuit = _circuit(api, cfg, n)
    obs = _observable(api, cfg, n, seed)
    if cfg == 5 and n == DEFAULT_QUBITS[5]:
        # BASELINE.json cfg 5: H must include qubits that sit on the shard index
        assert shard_flip_terms(obs, (30, 31, 32)) >= 1
    theta = np.random.default_rng([seed, cfg, 2]).uniform(0.0, 2.0 * np.pi, circuit.num_params)
    return Workload(cfg, n, circuit, obs, theta)
