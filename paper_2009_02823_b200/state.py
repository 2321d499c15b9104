"""Host-side state containers mirroring the reference ``StateVector`` API.

Mirrors ``svgrad/statevector.py:19-71`` (``StateVector``, ``init_basis_state``,
``clone_state``, ``inner_product``): complex128 amplitudes, little-endian
qubit order (qubit q is bit q of the amplitude index).  These are the
caller-facing inputs of the gradient call; the working states of the sweep
live in device memory owned by the native engine and never round-trip
through these objects.

``BasisState`` is the large-n fast path (SURVEY.md §7 "Host input states"):
it carries ``(num_qubits, basis_index)`` and only materialises the 2^n host
array if someone reads ``.amplitudes``, so a 33-qubit |0...0> input costs
nothing on the host and is initialised directly in HBM.
"""
from __future__ import annotations

import numpy as np


def _check_size(num_qubits: int) -> None:
    if num_qubits < 1:
        raise ValueError(f"need at least one qubit, got {num_qubits}")


class StateVector:
    """Dense complex128 amplitudes of a ``num_qubits`` register."""

    __slots__ = ("num_qubits", "amplitudes")

    def __init__(self, num_qubits: int, amplitudes):
        _check_size(num_qubits)
        amps = np.asarray(amplitudes, dtype=np.complex128)
        if amps.shape != (1 << num_qubits,):
            raise ValueError(
                f"expected {1 << num_qubits} amplitudes for {num_qubits} qubits, "
                f"got shape {amps.shape}"
            )
        self.num_qubits = num_qubits
        self.amplitudes = amps

    def norm(self) -> float:
        return float(np.linalg.norm(self.amplitudes))

    def __repr__(self) -> str:
        return f"StateVector(num_qubits={self.num_qubits})"


class BasisState:
    """Computational basis state |index> without a host-side 2^n array."""

    __slots__ = ("num_qubits", "basis_index", "_dense")

    def __init__(self, num_qubits: int, basis_index: int = 0):
        _check_size(num_qubits)
        if not 0 <= basis_index < (1 << num_qubits):
            raise ValueError(f"basis index {basis_index} out of range for {num_qubits} qubits")
        self.num_qubits = num_qubits
        self.basis_index = int(basis_index)
        self._dense = None

    @property
    def amplitudes(self) -> np.ndarray:
        if self._dense is None:
            amps = np.zeros(1 << self.num_qubits, dtype=np.complex128)
            amps[self.basis_index] = 1.0
            self._dense = amps
        return self._dense

    def norm(self) -> float:
        return 1.0

    def __repr__(self) -> str:
        return f"BasisState(num_qubits={self.num_qubits}, basis_index={self.basis_index})"


class ShardSlice:
    """This rank's slice of a ``num_qubits`` input state for a sharded NCCL engine.

    A rank of a job sharded over ``world`` GPUs by the top log2(world) qubits
    holds amplitudes ``rank * 2^m .. (rank + 1) * 2^m - 1`` (m = n - log2(world)).
    Passing this slice instead of the full StateVector keeps the host side of each
    rank at 16 * 2^m bytes (the reference's StateVector would be the whole 2^n
    array on every rank: 128 GiB at n = 33).  Same ``num_qubits`` semantics as
    StateVector; ``amplitudes`` is the local slice.
    """

    __slots__ = ("num_qubits", "amplitudes", "rank", "world")

    def __init__(self, num_qubits: int, amplitudes, rank: int, world: int):
        _check_size(num_qubits)
        if world < 1 or world & (world - 1) or not 0 <= rank < world or world > (1 << num_qubits):
            raise ValueError(f"bad rank {rank} / world {world} for {num_qubits} qubits")
        amps = np.asarray(amplitudes, dtype=np.complex128)
        local = (1 << num_qubits) // world
        if amps.shape != (local,):
            raise ValueError(f"expected {local} local amplitudes, got shape {amps.shape}")
        self.num_qubits = num_qubits
        self.amplitudes = amps
        self.rank = rank
        self.world = world

    def __repr__(self) -> str:
        return f"ShardSlice(num_qubits={self.num_qubits}, rank={self.rank}, world={self.world})"


def init_basis_state(num_qubits: int, basis_index: int = 0) -> StateVector:
    """|basis_index> as a dense StateVector (reference ``svgrad/statevector.py:43-53``)."""
    basis = BasisState(num_qubits, basis_index)
    return StateVector(num_qubits, basis.amplitudes)


def clone_state(src, counters=None) -> StateVector:
    if counters is not None:
        counters.clones += 1
    return StateVector(src.num_qubits, np.array(src.amplitudes, dtype=np.complex128, copy=True))


def inner_product(bra, ket, counters=None) -> complex:
    """<bra|ket>, conjugating the first argument."""
    if bra.num_qubits != ket.num_qubits:
        raise ValueError(f"qubit count mismatch: {bra.num_qubits} vs {ket.num_qubits}")
    if counters is not None:
        counters.inner_products += 1
    return complex(np.vdot(bra.amplitudes, ket.amplitudes))


def basis_index_of(state) -> int | None:
    """Basis index when ``state`` is known to be a basis state without scanning it."""
    if isinstance(state, BasisState):
        return state.basis_index
    return None
