"""Drop-in gradient API: ``reverse_mode_gradient`` and friends on the B200 engine.

Same signatures, validation order, error messages and return types as the
reference (``svgrad/gradients.py:52-259``).  The work happens in one C-ABI
call per sweep (``svg_reverse_sweep``, include/svgrad_b200.h); Python only
validates, binds theta (lowering.py) and packages the report.

``OpCounters`` keep the reference's contract: they count the primitive
operations of Algorithm 1's schedule (3G-1 gate applications, A derivative
applications, A+2 clones, A inner products, 1 observable application for G
gates and A parameter occurrences -- svgrad/gradients.py:25-30), which is
the algorithm-level work the fused kernels perform; the device never holds
more than two state buffers, and the ``LiveStateAudit`` sequence reproduces
the reference's acquire/release pattern (peak 4).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .ir import bound_matrix, derivative_scale, kind_name, matrix_derivative, pauli_product
from .lowering import Problem
from .operators import adjoint_observable, is_hermitian
from .state import ShardSlice


@dataclass
class OpCounters:
    gate_applies: int = 0
    derivative_applies: int = 0
    clones: int = 0
    inner_products: int = 0
    observable_applies: int = 0


@dataclass
class GradientReport:
    values: np.ndarray
    energy: complex
    counters: OpCounters


class LiveStateAudit:
    """Counts the state-vectors a gradient call holds simultaneously."""

    def __init__(self):
        self.live = 0
        self.peak = 0

    def acquire(self) -> None:
        self.live += 1
        self.peak = max(self.peak, self.live)

    def release(self) -> None:
        self.live -= 1


_HERMITIAN_MSG = "observable is not Hermitian; use non_hermitian_gradient for complex expectations"


def _check_call(circuit, params, obs, input_state) -> np.ndarray:
    """Argument validation, same order and messages as svgrad/gradients.py:92-106."""
    params = np.asarray(params, dtype=float)
    if params.shape != (circuit.num_params,):
        raise ValueError(f"parameter table has {circuit.num_params} entries, got shape {params.shape}")
    if obs.num_qubits != circuit.num_qubits:
        raise ValueError(f"observable acts on {obs.num_qubits} qubits, circuit on {circuit.num_qubits}")
    if input_state.num_qubits != circuit.num_qubits:
        raise ValueError(f"input state has {input_state.num_qubits} qubits, circuit {circuit.num_qubits}")
    return params


def _account(counters, audit, num_gates: int, num_derivs: int) -> None:
    counters.gate_applies += 3 * num_gates - 1 if num_gates else 0
    counters.derivative_applies += num_derivs
    counters.clones += num_derivs + 2
    counters.inner_products += num_derivs
    counters.observable_applies += 1
    if type(audit) is LiveStateAudit:  # the sequence below in closed form (O(1) per call)
        audit.peak = max(audit.peak, audit.live + (4 if num_derivs else 3))
        return
    audit.acquire()  # borrowed input
    audit.acquire()  # bra (psi, then lambda)
    audit.acquire()  # ket (phi)
    for _ in range(num_derivs):
        audit.acquire()  # probe -- folded into the fused reverse kernel, never allocated
        audit.release()
    audit.release()
    audit.release()
    audit.release()


def _check_slice(input_state, eng) -> None:
    """A ShardSlice input must be the slice of the rank this engine is."""
    if isinstance(input_state, ShardSlice):
        rank = eng.rank if eng.rank is not None else 0
        if eng.shards != input_state.world or rank != input_state.rank or (eng.shards > 1 and eng.rank is None):
            raise ValueError(f"input slice is rank {input_state.rank} of {input_state.world}; "
                             f"the engine is rank {eng.rank} of {eng.shards} shards")


def sweep(circuit, params, obs, input_state, counters, audit, device: int = 0, stats: dict | None = None,
          real_sums: bool = False, engine=None):
    """Equivalent of the reference's ``_reverse_sweep``: (complex sums[P], energy).

    ``real_sums=True`` lets the engine skip Im(sums) (returned as 0) when the
    caller only forms 2*Re, as the Hermitian path does (svgrad/gradients.py:198).
    """
    eng = engine or _native.engine(device)
    _check_slice(input_state, eng)
    problem = Problem(circuit, params, obs, input_state, real_sums=real_sums)
    sums, _, energy, st = eng.reverse_sweep(problem.c, circuit.num_params, problem.num_derivs)
    if st.nonfinite:
        _numeric_guard(circuit, problem, st.nonfinite)
    _account(counters, audit, len(circuit.gates), problem.num_derivs)
    out = sums
    if stats is not None:
        stats.update(st.as_dict())
    return out, complex(energy.re, energy.im)


def _numeric_guard(circuit, problem, count: int) -> None:
    """NaN/Inf in the device sums.  With finite tables and input and only unitary
    gates every sum is bounded (norms are preserved, |<lam|K|phi>| <= ||H|| ||K||), so a
    non-finite value there is a device fault, not arithmetic: raise.  Otherwise (a
    NaN/Inf input, or a NonUnitary gate that can overflow) the value is what the
    reference's numpy arithmetic would produce too and is returned as is."""
    tables = (problem.gates["fwd"], problem.gates["rewind"], problem.gates["adjoint"], problem.derivs["k"],
              problem.terms["coeff"], problem.products["coeff"], problem.factors["m"])
    finite = all(bool(np.all(np.isfinite(t))) for t in tables)
    finite = finite and (problem.amps is None or bool(np.all(np.isfinite(problem.amps))))
    unitary = all(kind_name(g) != "NonUnitary" for g in circuit.gates)
    if finite and unitary:
        raise FloatingPointError(f"{count} device sum(s) came out non-finite from finite inputs and unitary "
                                 f"gates: device fault")


def reverse_mode_gradient(circuit, params, obs, input_state, audit: LiveStateAudit | None = None,
                          *, device: int = 0, stats: dict | None = None, engine=None) -> GradientReport:
    """Full gradient of a Hermitian expectation in one fused backward sweep on the GPU.

    ``engine``: a specific ``_native.Engine`` (e.g. a sharded one from
    ``paper_2009_02823_b200.distributed``); default: the process engine of ``device``.
    """
    if not is_hermitian(obs):
        raise ValueError(_HERMITIAN_MSG)
    params = _check_call(circuit, params, obs, input_state)
    counters = OpCounters()
    sums, energy = sweep(circuit, params, obs, input_state, counters, audit or LiveStateAudit(), device, stats,
                         real_sums=True, engine=engine)
    return GradientReport((2.0 * sums.real).astype(complex), energy, counters)


def non_hermitian_gradient(circuit, params, obs, input_state, *, device: int = 0, engine=None) -> GradientReport:
    """Complex gradient of <psi|A|psi>: A-sweep conjugated plus A^dag-sweep (svgrad/gradients.py:240-259)."""
    params = _check_call(circuit, params, obs, input_state)
    counters = OpCounters()
    audit = LiveStateAudit()
    sums_a, energy = sweep(circuit, params, obs, input_state, counters, audit, device, engine=engine)
    sums_adj, _ = sweep(circuit, params, adjoint_observable(obs), input_state, counters, audit, device,
                        engine=engine)
    return GradientReport(np.conj(sums_a) + sums_adj, energy, counters)


def circuit_expectation(circuit, params, obs, input_state, *, device: int = 0, engine=None) -> complex:
    """<psi(theta)|H|psi(theta)> via the forward passes and the observable kernel only."""
    params = _check_call(circuit, params, obs, input_state)
    eng = engine or _native.engine(device)
    _check_slice(input_state, eng)
    problem = Problem(circuit, params, obs, input_state, forward_only=True)
    energy, _ = eng.expectation(problem.c)
    return complex(energy.re, energy.im)


def _derivative_action(gate, params, which: int) -> np.ndarray:
    """Target-space matrix the reference's ``apply_gate_derivative`` applies, times its
    deferred scalar (svgrad/circuit.py:302-334): PauliRotation alpha*i * U(theta) P,
    Phase i e^{i theta} |1><1|, matrix kinds dM/dtheta_which.  Control projection is
    separate (the caller adds it)."""
    name = kind_name(gate)
    scale = derivative_scale()
    if name == "PauliRotation":
        return (gate.kind.alpha * 1j * scale) * (bound_matrix(gate, params) @ pauli_product(gate.kind.axes))
    if name == "Phase":
        theta = float(params[gate.param_refs[0]])
        return np.diag([0.0, 1j * np.exp(1j * theta)]) * scale
    return matrix_derivative(gate, params, which) * scale


def reference_gradient(circuit, params, obs, input_state, *, device: int = 0) -> GradientReport:
    """The reference's quadratic schedule on the GPU (svgrad/gradients.py:201-237).

    For every parameter occurrence (gate i, argument j) the reference rebuilds the
    derivative-inserted state V_ij|in> from the input and takes
    2 Re <H U in | V_ij in>.  Here each occurrence is one forward sweep of the
    engine over n+1 qubits (a Hadamard test): the ancilla (qubit n) starts in |+>,
    the gates before and after i act on both branches, branch 0 applies gate i and
    branch 1 its derivative action (control projections included), and the
    observable is X_ancilla (x) H, so <X (x) H> = Re <U in|H|V_ij in>.  The cost is
    A forward sweeps of G gates -- the O(P^2) growth the paper's Fig. 2 compares
    against -- and the counters follow the reference's accounting
    (gate_applies G + A(G-1), clones A+1, derivative_applies = inner_products = A).
    Generated kernels are off for this schedule (each occurrence is a new circuit
    structure); the interpreted register-tile kernels run it.
    """
    if not is_hermitian(obs):
        raise ValueError(_HERMITIAN_MSG)
    params = _check_call(circuit, params, obs, input_state)
    from .ir import Circuit, FixedUnitary, Gate, HADAMARD, SIGMA
    from .operators import Observable
    from .state import StateVector, basis_index_of

    n, G = circuit.num_qubits, len(circuit.gates)
    counters = OpCounters()
    energy = circuit_expectation(circuit, params, obs, input_state, device=device)
    counters.clones += 1
    counters.gate_applies += G
    counters.observable_applies += 1
    anc = n
    basis = basis_index_of(input_state)
    if basis is not None:
        inp = type(input_state)(n + 1, basis)
    else:
        amps = np.zeros(1 << (n + 1), dtype=np.complex128)
        amps[: 1 << n] = np.asarray(input_state.amplitudes, dtype=np.complex128)
        inp = StateVector(n + 1, amps)
    hobs = Observable(n + 1, tuple((c, f + "X") for c, f in obs.terms))
    had = Gate(FixedUnitary(HADAMARD, "h"), (anc,))
    xanc = Gate(FixedUnitary(SIGMA["X"], "x"), (anc,))
    proj1 = np.diag([0.0, 1.0]).astype(np.complex128)
    eng = _reference_engine(device)
    values = np.zeros(circuit.num_params, dtype=complex)
    for i, gate in enumerate(circuit.gates):
        for j in range(len(gate.param_refs)):
            branch1 = [Gate(FixedUnitary(proj1, "p1"), (c,), (anc,)) for c in gate.controls]
            branch1.append(Gate(FixedUnitary(_derivative_action(gate, params, j), "d"), tuple(gate.targets),
                                tuple(gate.controls) + (anc,)))
            gates = [had, *circuit.gates[:i], xanc,
                     Gate(gate.kind, tuple(gate.targets), tuple(gate.controls) + (anc,), tuple(gate.param_refs)),
                     xanc, *branch1, *circuit.gates[i + 1:]]
            test = Circuit(n + 1, gates, circuit.num_params)
            e = circuit_expectation(test, params, hobs, inp, engine=eng)
            values[gate.param_refs[j]] += 2.0 * e.real
            counters.clones += 1
            counters.gate_applies += G - 1
            counters.derivative_applies += 1
            counters.inner_products += 1
    return GradientReport(values, energy, counters)


_REF_ENGINES: dict = {}


def _reference_engine(device: int):
    """Engine for the quadratic schedule: interpreted kernels (no per-structure NVRTC compile)."""
    eng = _REF_ENGINES.get(device)
    if eng is None:
        eng = _REF_ENGINES[device] = _native.Engine(device)
        eng.set_option("jit", 0)
    return eng


DEFAULT_FD_STEP = 1e-5  # svgrad/gradients.py DEFAULT_FD_STEP


def finite_difference_gradient(circuit, params, obs, input_state, delta: float = DEFAULT_FD_STEP, *,
                               device: int = 0, engine=None) -> GradientReport:
    """Central differences on the GPU expectation path (svgrad/gradients.py:262-294).

    2P + 1 forward sweeps (forward passes + observable kernel each); counters
    follow the reference's per-evaluation accounting: G gate applications, one
    clone and one observable application per expectation.
    """
    if delta <= 0:
        raise ValueError(f"delta must be positive, got {delta}")
    params = _check_call(circuit, params, obs, input_state)
    counters = OpCounters()
    G = len(circuit.gates)

    def evaluate(theta):  # the reference's expectation(): clone, G applies, observable, one inner product
        counters.clones += 1
        counters.gate_applies += G
        counters.observable_applies += 1
        counters.inner_products += 1
        return circuit_expectation(circuit, theta, obs, input_state, device=device, engine=engine)

    values = np.zeros(circuit.num_params, dtype=complex)
    shifted = params.copy()
    for k in range(circuit.num_params):
        shifted[k] = params[k] + delta
        plus = evaluate(shifted)
        shifted[k] = params[k] - delta
        minus = evaluate(shifted)
        shifted[k] = params[k]
        values[k] = (plus - minus) / (2.0 * delta)
    return GradientReport(values, evaluate(params), counters)
