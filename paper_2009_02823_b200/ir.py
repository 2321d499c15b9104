"""Circuit IR mirroring the reference types, plus host-side binding.

Same names, fields and validation as the reference (``svgrad/circuit.py:43-219``):
gate kinds ``PauliRotation`` / ``Phase`` / ``FixedUnitary`` / ``CustomParametric`` /
``NonUnitary``, ``Gate(kind, targets, controls, param_refs)``,
``Circuit(num_qubits, gates, num_params)`` and the factories ``rx ry rz rp
phase_gate fixed cx crx cry crz``.  Reference objects are accepted too: every
consumer in this package reads gates through the duck-typed accessors at the
bottom (kind recognised by class name), never through ``isinstance``.

Binding (theta -> small matrices) happens here on the host, once per call,
exactly like ``_bind`` (``svgrad/gradients.py:109-111``); the device only
ever sees bound coefficients.
"""
from __future__ import annotations

import contextlib
import sys
from dataclasses import dataclass
from typing import Callable, Union

import numpy as np

ENTRY_DERIV_STEP = 1e-6  # central-difference step, svgrad/circuit.py:28
PIVOT_EPS = 1e-14        # singularity threshold, svgrad/gates.py:10

SIGMA = {
    "I": np.eye(2, dtype=np.complex128),
    "X": np.array([[0, 1], [1, 0]], dtype=np.complex128),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    "Z": np.array([[1, 0], [0, -1]], dtype=np.complex128),
}
HADAMARD = np.array([[1, 1], [1, -1]], dtype=np.complex128) / np.sqrt(2.0)
NAMED_FIXED = {"h": HADAMARD, "x": SIGMA["X"], "y": SIGMA["Y"], "z": SIGMA["Z"]}


class NonInvertibleGateError(ValueError):
    """A gate whose bound matrix cannot be inverted, named by circuit index."""


# -- gate kinds ----------------------------------------------------------------------

@dataclass(frozen=True)
class PauliRotation:
    """exp(alpha * i * theta * P), P a product of one Pauli per target."""

    axes: str
    alpha: float = -0.5

    def __post_init__(self):
        if not self.axes or set(self.axes) - set("XYZ"):
            raise ValueError(f"axes must be a nonempty string over XYZ, got {self.axes!r}")

    @property
    def arity(self) -> int:
        return 1


@dataclass(frozen=True)
class Phase:
    """diag(1, e^{i theta}) on one target."""

    @property
    def arity(self) -> int:
        return 1


@dataclass(frozen=True, eq=False)
class FixedUnitary:
    matrix: np.ndarray
    name: str = ""

    @property
    def arity(self) -> int:
        return 0

    def __eq__(self, other):
        if not isinstance(other, FixedUnitary):
            return NotImplemented
        return self.name == other.name and np.array_equal(self.matrix, other.matrix)


@dataclass(frozen=True, eq=False)
class CustomParametric:
    matrix_fn: Callable[..., np.ndarray]
    num_params: int = 1
    derivative_fn: Callable[..., np.ndarray] | None = None
    name: str = ""

    @property
    def arity(self) -> int:
        return self.num_params


@dataclass(frozen=True, eq=False)
class NonUnitary:
    matrix_fn: Callable[..., np.ndarray]
    num_params: int = 0
    derivative_fn: Callable[..., np.ndarray] | None = None
    invertible: bool = True
    name: str = ""

    @property
    def arity(self) -> int:
        return self.num_params


GateKind = Union[PauliRotation, Phase, FixedUnitary, CustomParametric, NonUnitary]


@dataclass(frozen=True)
class Gate:
    kind: GateKind
    targets: tuple[int, ...]
    controls: tuple[int, ...] = ()
    param_refs: tuple[int, ...] = ()

    def __post_init__(self):
        for field in ("targets", "controls", "param_refs"):
            object.__setattr__(self, field, tuple(getattr(self, field)))
        t, c = self.targets, self.controls
        if set(t) & set(c):
            raise ValueError(f"targets {t} and controls {c} overlap")
        if len(set(t)) != len(t):
            raise ValueError(f"duplicate targets in {t}")
        if len(self.param_refs) != self.kind.arity:
            raise ValueError(
                f"{type(self.kind).__name__} consumes {self.kind.arity} parameter(s), "
                f"got refs {self.param_refs}"
            )
        if isinstance(self.kind, PauliRotation) and len(self.kind.axes) != len(t):
            raise ValueError(f"axes {self.kind.axes!r} need {len(self.kind.axes)} targets, got {t}")
        if isinstance(self.kind, Phase) and len(t) != 1:
            raise ValueError(f"phase gates act on one target, got {t}")
        if len(t) not in (1, 2):
            raise ValueError(f"gates act on 1 or 2 targets, got {t}")


@dataclass(frozen=True)
class Circuit:
    num_qubits: int
    gates: tuple[Gate, ...]
    num_params: int

    def __post_init__(self):
        object.__setattr__(self, "gates", tuple(self.gates))
        for i, gate in enumerate(self.gates):
            for q in (*gate.targets, *gate.controls):
                if not 0 <= q < self.num_qubits:
                    raise ValueError(f"gate {i}: qubit {q} out of range")
            for p in gate.param_refs:
                if not 0 <= p < self.num_params:
                    raise ValueError(f"gate {i}: parameter index {p} out of range")


# -- factories (svgrad/circuit.py:179-216) ---------------------------------------------

def rx(target: int, param: int, alpha: float = -0.5) -> Gate:
    return Gate(PauliRotation("X", alpha), (target,), (), (param,))


def ry(target: int, param: int, alpha: float = -0.5) -> Gate:
    return Gate(PauliRotation("Y", alpha), (target,), (), (param,))


def rz(target: int, param: int, alpha: float = -0.5) -> Gate:
    return Gate(PauliRotation("Z", alpha), (target,), (), (param,))


def rp(axes: str, targets, param: int, alpha: float = -0.5) -> Gate:
    return Gate(PauliRotation(axes.upper(), alpha), tuple(targets), (), (param,))


def phase_gate(target: int, param: int) -> Gate:
    return Gate(Phase(), (target,), (), (param,))


def fixed(name: str, target: int) -> Gate:
    return Gate(FixedUnitary(NAMED_FIXED[name], name), (target,), (), ())


def cx(control: int, target: int) -> Gate:
    return Gate(FixedUnitary(SIGMA["X"], "x"), (target,), (control,), ())


def crx(control: int, target: int, param: int, alpha: float = -0.5) -> Gate:
    return Gate(PauliRotation("X", alpha), (target,), (control,), (param,))


def cry(control: int, target: int, param: int, alpha: float = -0.5) -> Gate:
    return Gate(PauliRotation("Y", alpha), (target,), (control,), (param,))


def crz(control: int, target: int, param: int, alpha: float = -0.5) -> Gate:
    return Gate(PauliRotation("Z", alpha), (target,), (control,), (param,))


# -- negative-control hook (svgrad/circuit.py:286-299) ------------------------------------

_DERIV_SCALE = 1.0


@contextlib.contextmanager
def perturbed_derivative_scale(scale: float):
    """Scale every derivative generator; the selftest's negative control."""
    global _DERIV_SCALE
    saved, _DERIV_SCALE = _DERIV_SCALE, float(scale)
    try:
        yield
    finally:
        _DERIV_SCALE = saved


def derivative_scale() -> float:
    """Current generator scale; also honours the reference's own hook if the
    caller already imported it (drop-in use under the reference's selftest)."""
    ref = sys.modules.get("svgrad.circuit")
    ref_scale = float(getattr(ref, "_DERIV_SCALE", 1.0)) if ref is not None else 1.0
    return _DERIV_SCALE * ref_scale


# -- duck-typed access (reference objects or ours) -----------------------------------------

def kind_name(gate) -> str:
    return type(gate.kind).__name__


def pauli_product(axes: str) -> np.ndarray:
    """Kronecker product with axes[k] on bit k of the joint index (little-endian)."""
    out = SIGMA[axes[0]]
    for a in axes[1:]:
        out = np.kron(SIGMA[a], out)
    return out


def invert_small(m: np.ndarray) -> np.ndarray:
    """2x2 analytic / 4x4 partial-pivot inverse with the reference's singularity rule.

    Same thresholds and messages as ``svgrad/gates.py:58-79``.
    """
    m = np.asarray(m, dtype=np.complex128)
    if m.shape == (2, 2):
        det = m[0, 0] * m[1, 1] - m[0, 1] * m[1, 0]
        if abs(det) <= PIVOT_EPS:
            raise ValueError(f"singular 2x2 matrix (|det| = {abs(det):.3e})")
        return np.array([[m[1, 1], -m[0, 1]], [-m[1, 0], m[0, 0]]]) / det
    if m.shape == (4, 4):
        a = m.copy()
        inv = np.eye(4, dtype=np.complex128)
        min_pivot = np.inf
        for col in range(4):
            piv = col + int(np.argmax(np.abs(a[col:, col])))
            min_pivot = min(min_pivot, abs(a[piv, col]))
            if piv != col:
                a[[col, piv]] = a[[piv, col]]
                inv[[col, piv]] = inv[[piv, col]]
            if abs(a[col, col]) <= PIVOT_EPS:
                continue
            f = a[col + 1:, col] / a[col, col]
            a[col + 1:] -= np.outer(f, a[col])
            inv[col + 1:] -= np.outer(f, inv[col])
        if min_pivot <= PIVOT_EPS:
            raise ValueError(f"singular 4x4 matrix (min pivot = {min_pivot:.3e})")
        for col in range(3, -1, -1):
            inv[col] /= a[col, col]
            a[col] /= a[col, col]
            inv[:col] -= np.outer(a[:col, col], inv[col])
            a[:col] -= np.outer(a[:col, col], a[col])
        return inv
    raise ValueError(f"expected a 2x2 or 4x4 matrix, got shape {m.shape}")


def bound_matrix(gate, params) -> np.ndarray:
    """Target-space matrix at theta (``gate_matrix``, svgrad/circuit.py:228-243)."""
    kind, name = gate.kind, kind_name(gate)
    if name == "PauliRotation":
        ang = kind.alpha * float(params[gate.param_refs[0]])
        p = pauli_product(kind.axes)
        return np.cos(ang) * np.eye(p.shape[0]) + 1j * np.sin(ang) * p
    if name == "Phase":
        return np.array([[1, 0], [0, np.exp(1j * float(params[gate.param_refs[0]]))]], dtype=np.complex128)
    if name == "FixedUnitary":
        return np.asarray(kind.matrix, dtype=np.complex128)
    m = np.asarray(kind.matrix_fn(*[float(params[k]) for k in gate.param_refs]), dtype=np.complex128)
    dim = 1 << len(gate.targets)
    if m.shape != (dim, dim):
        raise ValueError(f"matrix function returned shape {m.shape} for {len(gate.targets)} targets")
    return m


def matrix_derivative(gate, params, which: int) -> np.ndarray:
    """d(matrix)/d(angle_which) for the callable kinds: analytic or central FD."""
    kind = gate.kind
    values = [float(params[k]) for k in gate.param_refs]
    if kind.derivative_fn is not None:
        return np.asarray(kind.derivative_fn(which, *values), dtype=np.complex128)
    hi, lo = list(values), list(values)
    hi[which] += ENTRY_DERIV_STEP
    lo[which] -= ENTRY_DERIV_STEP
    m_hi = np.asarray(kind.matrix_fn(*hi), dtype=np.complex128)
    m_lo = np.asarray(kind.matrix_fn(*lo), dtype=np.complex128)
    return (m_hi - m_lo) / (2 * ENTRY_DERIV_STEP)
