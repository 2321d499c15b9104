"""Observables (sums of tensor-product terms) and their Pauli lowering.

``Observable`` mirrors ``svgrad/observable.py:42-76``: terms are
``(coefficient, factor_string)`` with letters ``I X Y Z H + -`` and string
position j acting on qubit j; ``is_hermitian`` uses the same structural rule
and the same dense fallback for at most 10 qubits.

For the device a term is lowered to Pauli strings ``(c, x_mask, z_mask,
n_y)`` -- ``H = (X+Z)/sqrt2``, ``+ = (X - iY)/2``, ``- = (X + iY)/2`` expand
a term with w such letters into 2^w strings -- when w <= 3, and otherwise kept
as a product of 2x2 factor matrices (product-term passes on the device, e.g.
the paper's benchmark operator ``hadamard_all`` as Walsh-Hadamard butterflies).
A Pauli string P acts as ``(P psi)[m] = i^{n_y} (-1)^{popcount((m^x) & z)} psi[m ^ x]``
with ``x`` = qubits holding X or Y and ``z`` = qubits holding Z or Y.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property
from itertools import product

import numpy as np

from .ir import HADAMARD, SIGMA

LETTERS = "IXYZH+-"
FACTOR_MATRICES = {
    **SIGMA,
    "H": HADAMARD,
    "+": np.array([[0, 0], [1, 0]], dtype=np.complex128),
    "-": np.array([[0, 1], [0, 0]], dtype=np.complex128),
}
_ADJOINT = str.maketrans("+-", "-+")
_DENSE_HERMITICITY_MAX_QUBITS = 10
# Expansion of non-Pauli letters into Pauli strings: letter -> [(weight, pauli)]
_EXPANSION = {
    "I": ((1.0, "I"),),
    "X": ((1.0, "X"),),
    "Y": ((1.0, "Y"),),
    "Z": ((1.0, "Z"),),
    "H": ((1.0 / np.sqrt(2.0), "X"), (1.0 / np.sqrt(2.0), "Z")),
    "+": ((0.5, "X"), (-0.5j, "Y")),
    "-": ((0.5, "X"), (0.5j, "Y")),
}
# Terms with more than this many H/+/- letters stay products of 2x2 factors on
# the device (product-term passes: Walsh-Hadamard butterflies for H) instead of
# 2^w Pauli strings; the observable passes share one partner load per flip mask,
# so a few strings are cheaper than a product pipeline's extra state passes.
MAX_EXPANDED_LETTERS = 3


@dataclass(frozen=True)
class Observable:
    num_qubits: int
    terms: tuple[tuple[complex, str], ...]

    def __post_init__(self):
        object.__setattr__(self, "terms", tuple((complex(c), str(f)) for c, f in self.terms))
        if not self.terms:
            raise ValueError("an observable needs at least one term")
        for _, factors in self.terms:
            if len(factors) != self.num_qubits:
                raise ValueError(f"factor string {factors!r} does not cover {self.num_qubits} qubits")
            bad = set(factors) - set(LETTERS)
            if bad:
                raise ValueError(f"unknown factor letter {sorted(bad)[0]!r} in {factors!r}")

    @property
    def num_terms(self) -> int:
        return len(self.terms)

    @cached_property
    def is_hermitian(self) -> bool:
        return hermitian(self)


def hermitian(obs) -> bool:
    """Structural rule, else dense check up to 10 qubits (svgrad/observable.py:66-76)."""
    if all(complex(c).imag == 0.0 and "+" not in f and "-" not in f for c, f in obs.terms):
        return True
    if obs.num_qubits > _DENSE_HERMITICITY_MAX_QUBITS:
        return False
    m = dense_matrix(obs)
    return bool(np.allclose(m, m.conj().T, atol=1e-12))


def is_hermitian(obs) -> bool:
    flag = getattr(obs, "is_hermitian", None)
    return bool(flag) if flag is not None else hermitian(obs)


def dense_matrix(obs) -> np.ndarray:
    """2^N x 2^N matrix, for small checks only."""
    dim = 1 << obs.num_qubits
    out = np.zeros((dim, dim), dtype=np.complex128)
    for coeff, factors in obs.terms:
        term = FACTOR_MATRICES[factors[0]]
        for ch in factors[1:]:
            term = np.kron(FACTOR_MATRICES[ch], term)
        out += complex(coeff) * term
    return out


def adjoint_observable(obs) -> Observable:
    """Term-wise adjoint: conjugate coefficients, swap + and - (svgrad/observable.py:103-111)."""
    return Observable(
        obs.num_qubits,
        tuple((complex(c).conjugate(), f.translate(_ADJOINT)) for c, f in obs.terms),
    )


def builtin_observable(name: str, num_qubits: int) -> Observable:
    if name == "hadamard_all":
        return Observable(num_qubits, ((1.0, "H" * num_qubits),))
    if name == "z_all":
        return Observable(num_qubits, ((1.0, "Z" * num_qubits),))
    raise ValueError(f"unknown builtin observable {name!r}")


BUILTIN_OBSERVABLES = ("hadamard_all", "z_all")


@dataclass(frozen=True)
class PauliString:
    coeff: complex
    x_mask: int
    z_mask: int
    n_y: int


def pauli_masks(letters: str) -> tuple[int, int, int]:
    x = z = ny = 0
    for q, ch in enumerate(letters):
        if ch in "XY":
            x |= 1 << q
        if ch in "ZY":
            z |= 1 << q
        ny += ch == "Y"
    return x, z, ny


def split_terms(obs, max_letters: int = MAX_EXPANDED_LETTERS):
    """(terms for the Pauli expansion, terms kept as 2x2-factor products), in term order."""
    pauli, prods = [], []
    for coeff, factors in obs.terms:
        wide = sum(ch in "H+-" for ch in factors) > max_letters
        (prods if wide else pauli).append((complex(coeff), factors))
    return tuple(pauli), tuple(prods)


def pauli_strings(obs, limit: int | None = None) -> list[PauliString]:
    """Expand every term into Pauli strings, in term order (no merging).
    ``limit``: refuse expansions wider than this (None: no limit)."""
    out: list[PauliString] = []
    for coeff, factors in obs.terms:
        coeff = complex(coeff)
        if set(factors) <= set("IXYZ"):
            out.append(PauliString(coeff, *pauli_masks(factors)))
            continue
        choices = [_EXPANSION[ch] for ch in factors]
        width = 1
        for c in choices:
            width *= len(c)
        if limit is not None and len(out) + width > limit:
            raise ValueError(f"term {factors!r} expands to {width} Pauli strings (limit {limit})")
        for combo in product(*choices):
            w = coeff
            for weight, _ in combo:
                w *= weight
            out.append(PauliString(w, *pauli_masks("".join(p for _, p in combo))))
    return out
