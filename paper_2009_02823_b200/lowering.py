"""Host lowering: (circuit, theta, observable, input) -> svg_problem tables.

This is the reference's binding step (``_bind`` / ``_rewind_matrices`` /
deferred derivative scalars, svgrad/gradients.py:109-125 and
svgrad/circuit.py:228-334) restated as flat, device-ready tables:

* Pauli-form gates (every ``PauliRotation``, and ``FixedUnitary`` X/Y/Z incl.
  CX/CY/CZ) become ``op = a*I + b*P`` with the gate's Pauli product P:
  ``U = cos(alpha*theta) I + i sin(alpha*theta) P`` (svgrad/gates.py:42-50),
  ``U^-1 = U^dag = conj(a) I + conj(b) P``, and the derivative generator in
  the post-gate basis (svg_deriv.basis = 1), ``K' = alpha*i * P``: the
  reference's probe is ``alpha*i * U P phi_i = alpha*i * P phi_{i+1}``
  (it applies P then U and defers alpha*i, svgrad/circuit.py:316-321).
* Dense-matrix gates (``Phase``, other ``FixedUnitary``, ``CustomParametric``,
  ``NonUnitary``) ship U, the rewind (adjoint, or the true inverse for
  NonUnitary -> ``NonInvertibleGateError`` text identical to
  svgrad/gradients.py:121-122) and U^dag, plus K = scalar * dU/dtheta_j
  (Phase: i e^{i theta} |1><1|; matrix kinds: analytic or central-FD dM).
* Control projection (svgrad/circuit.py:330-331) is the gate's ctrl mask:
  the device evaluates K only where every control bit is 1.

The theta-independent structure of a circuit is cached per circuit object,
so a VQE loop re-binds only the coefficient arrays.
"""
from __future__ import annotations

import ctypes as C
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .ir import NonInvertibleGateError, SIGMA, bound_matrix, derivative_scale, invert_small, kind_name, matrix_derivative
from .operators import FACTOR_MATRICES, pauli_masks, pauli_strings, split_terms
from .state import ShardSlice, basis_index_of

GATE_DTYPE = np.dtype(  # itemsize 816 = 51 complex128 slots (bind scatters into a flat complex view)
    [
        ("form", "<i4"), ("ntargets", "<i4"), ("targets", "<i4", (2,)), ("ctrl_mask", "<u8"),
        ("x_mask", "<u8"), ("z_mask", "<u8"), ("n_y", "<i4"), ("nderiv", "<i4"),
        ("fwd", "<c16", (16,)), ("rewind", "<c16", (16,)), ("adjoint", "<c16", (16,)),
    ],
    align=True,
)
DERIV_DTYPE = np.dtype(
    [("gate", "<i4"), ("param_ref", "<i4"), ("form", "<i4"), ("basis", "<i4"), ("k", "<c16", (16,))],
    align=True,
)
TERM_DTYPE = np.dtype(
    [("coeff", "<c16"), ("x_mask", "<u8"), ("z_mask", "<u8"), ("n_y", "<i4"), ("reserved", "<i4")],
    align=True,
)
PRODUCT_DTYPE = np.dtype([("coeff", "<c16"), ("first_factor", "<i4"), ("num_factors", "<i4")], align=True)
FACTOR_DTYPE = np.dtype([("qubit", "<i4"), ("reserved", "<i4"), ("m", "<c16", (4,))], align=True)
_PAULI_FIXED = {"X": SIGMA["X"], "Y": SIGMA["Y"], "Z": SIGMA["Z"]}
FLAG_REAL_SUMS = 1  # SVG_FLAG_REAL_SUMS: only 2*Re(sums) is consumed (Hermitian observables)
FLAG_INPUT_LOCAL = 2  # SVG_FLAG_INPUT_LOCAL: input_amps is this rank's shard slice (state.ShardSlice)


@dataclass
class Structure:
    """theta-independent part of a lowered circuit."""

    gates: np.ndarray            # GATE_DTYPE, masks/targets filled, coefficients zero
    derivs: np.ndarray           # DERIV_DTYPE, gate/param_ref/form filled
    rot_gates: np.ndarray        # indices of PauliRotation gates
    rot_refs: np.ndarray         # their parameter slot
    rot_alpha: np.ndarray        # their alpha
    rot_derivs: np.ndarray       # their derivative row
    fixed_pauli: np.ndarray      # indices of X/Y/Z fixed gates (a=0, b=1)
    mat_gates: list              # indices of dense-matrix gates (bound per call)
    num_derivs: int


_cache: dict[int, tuple] = {}
_tls = threading.local()


def _structure(circuit) -> Structure:
    hit = _cache.get(id(circuit))
    if hit is not None and hit[0]() is circuit:
        return hit[1]
    gates = circuit.gates
    G = len(gates)
    arr = np.zeros(G, dtype=GATE_DTYPE)
    rot_g, rot_r, rot_a, rot_d, fixed_p, mats = [], [], [], [], [], []
    drows = []
    for i, g in enumerate(gates):
        name = kind_name(g)
        targets = tuple(g.targets)
        ctrl = 0
        for c in g.controls:
            ctrl |= 1 << c
        rec = arr[i]
        rec["ntargets"] = len(targets)
        rec["targets"][: len(targets)] = targets
        rec["ctrl_mask"] = ctrl
        arity = len(g.param_refs)
        rec["nderiv"] = arity
        form = N.FORM_MAT
        if name == "PauliRotation":
            form = N.FORM_PAULI
            letters = ["I"] * (max(targets) + 1)
            for axis, t in zip(g.kind.axes, targets):
                letters[t] = axis
            x, z, ny = pauli_masks("".join(letters))
            rec["x_mask"], rec["z_mask"], rec["n_y"] = x, z, ny
            rot_g.append(i)
            rot_r.append(g.param_refs[0])
            rot_a.append(float(g.kind.alpha))
            rot_d.append(len(drows))
        elif name == "FixedUnitary" and len(targets) == 1:
            m = np.asarray(g.kind.matrix, dtype=np.complex128)
            axis = next((a for a, s in _PAULI_FIXED.items() if m.shape == (2, 2) and np.array_equal(m, s)), None)
            if axis is not None:
                form = N.FORM_PAULI
                x, z, ny = pauli_masks("I" * targets[0] + axis)
                rec["x_mask"], rec["z_mask"], rec["n_y"] = x, z, ny
                fixed_p.append(i)
        rec["form"] = form
        if form == N.FORM_MAT:
            mats.append(i)
        for j in range(arity):
            drows.append((i, g.param_refs[j], form))
    derivs = np.zeros(len(drows), dtype=DERIV_DTYPE)
    if drows:
        d = np.asarray(drows, dtype=np.int64)
        derivs["gate"], derivs["param_ref"], derivs["form"] = d[:, 0], d[:, 1], d[:, 2]
    st = Structure(
        arr, derivs, np.asarray(rot_g, dtype=np.int64), np.asarray(rot_r, dtype=np.int64),
        np.asarray(rot_a, dtype=np.float64), np.asarray(rot_d, dtype=np.int64),
        np.asarray(fixed_p, dtype=np.int64), mats, len(drows),
    )
    try:
        ref = weakref.ref(circuit)
    except TypeError:  # not weak-referenceable: do not cache
        return st
    if len(_cache) > 64:
        _cache.clear()
    _cache[id(circuit)] = (ref, st)
    return st


def _put(block: np.ndarray, m: np.ndarray) -> None:
    flat = np.asarray(m, dtype=np.complex128).reshape(-1)
    block[:] = 0
    block[: flat.size] = flat


def bind(circuit, params: np.ndarray, forward_only: bool = False) -> tuple[np.ndarray, np.ndarray]:
    """Gate and derivative tables for one theta (raises NonInvertibleGateError).

    ``forward_only``: the tables feed a forward sweep only (expectation), which never
    rewinds -- a singular NonUnitary gate is accepted there, as in the reference's
    forward-only paths (svgrad/gradients.py:201-237, 262-294)."""
    st = _structure(circuit)
    # per-thread working tables, reused across calls (every theta-dependent field
    # is rewritten below; the rest is structure): no 100s-of-KB copy per call
    tls = _tls.__dict__.setdefault("tables", {})
    hit = tls.get(id(st))
    if hit is None or hit[0] is not st:
        if len(tls) > 16:
            tls.clear()
        g, d = st.gates.copy(), st.derivs.copy()
        # the rotation coefficients a = cos, b = i sin of (fwd, rewind, adjoint) as
        # positions in a flat float64 view of the gate records (imag(a) = re(b) = 0
        # from the structure): three scatters per call, no temporaries
        fl = g.view(np.float64).reshape(-1)
        base = st.rot_gates * (GATE_DTYPE.itemsize // 8)
        off = {f: GATE_DTYPE.fields[f][1] // 8 for f in ("fwd", "rewind", "adjoint")}
        re_a = np.stack([base + off[f] for f in ("fwd", "rewind", "adjoint")])   # real(a), 3 x nrot
        im_b = base + off["fwd"] + 3                                              # imag(b) of U
        im_bc = np.stack([base + off[f] + 3 for f in ("rewind", "adjoint")])     # imag(b) of U^dag
        for field in ("fwd", "rewind", "adjoint"):  # fixed X/Y/Z: a = 0, b = 1
            g[field][st.fixed_pauli, 1] = 1.0
        d["basis"][st.rot_derivs] = 1  # rotation generators in the post-gate basis
        hit = tls[id(st)] = [st, g, d, fl, re_a, im_b, im_bc, d["k"], None]
    _, gates, derivs, fl, re_a, im_b, im_bc, dk, last_scale = hit
    scale = derivative_scale()
    if st.rot_gates.size:
        ang = st.rot_alpha * params[st.rot_refs]
        c, sn = np.cos(ang), np.sin(ang)
        fl[re_a] = c
        fl[im_b] = sn
        np.negative(sn, out=sn)
        fl[im_bc] = sn
        if scale != last_scale:
            # post-gate generator (basis 1): dU phi_i = alpha*i P U phi_i = alpha*i P phi_{i+1}
            dk[st.rot_derivs, 1] = (st.rot_alpha * 1j) * scale
            hit[8] = scale
    if st.mat_gates:
        first = np.concatenate([[0], np.cumsum(gates["nderiv"])])
        for i in st.mat_gates:
            g = circuit.gates[i]
            name = kind_name(g)
            m = bound_matrix(g, params)
            adj = m.conj().T
            if name == "NonUnitary":
                try:
                    rew = invert_small(m)
                except ValueError as exc:
                    if not forward_only:
                        raise NonInvertibleGateError(f"non-invertible gate {i}: {exc}") from exc
                    rew = adj  # never read: no rewind in a forward sweep
            else:
                rew = adj
            _put(gates["fwd"][i], m)
            _put(gates["rewind"][i], rew)
            _put(gates["adjoint"][i], adj)
            for j in range(len(g.param_refs)):
                if name == "Phase":
                    theta = float(params[g.param_refs[0]])
                    k = np.diag([0.0, 1j * np.exp(1j * theta)])
                else:
                    k = matrix_derivative(g, params, j)
                _put(derivs["k"][first[i] + j], k * scale)
    return gates, derivs


def _lower_terms(obs):
    """(Pauli-string table, product-term table, factor table) of an observable:
    terms with at most a few H/+/- letters are expanded into Pauli strings, wider
    ones stay products of 2x2 factors (operators.split_terms)."""
    pauli_terms, products = split_terms(obs)
    strings = pauli_strings(type("T", (), {"terms": pauli_terms})()) if pauli_terms else []
    terms = np.zeros(len(strings), dtype=TERM_DTYPE)
    for i, s in enumerate(strings):
        terms[i] = (s.coeff, s.x_mask, s.z_mask, s.n_y, 0)
    nf = sum(sum(ch != "I" for ch in f) for _, f in products)
    prods = np.zeros(len(products), dtype=PRODUCT_DTYPE)
    factors = np.zeros(nf, dtype=FACTOR_DTYPE)
    j = 0
    for i, (c, f) in enumerate(products):
        first = j
        for q, ch in enumerate(f):
            if ch != "I":
                factors[j] = (q, 0, FACTOR_MATRICES[ch].reshape(-1))
                j += 1
        prods[i] = (complex(c), first, j - first)
    return terms, prods, factors


_TERMS_CACHE: dict = {}


def lower_terms(obs):
    """(Pauli strings, product terms, factors) tables, cached per observable terms
    object (terms are immutable tuples: a repeated gradient call on the same
    observable reuses them)."""
    terms_obj = obs.terms
    hit = _TERMS_CACHE.get(id(terms_obj))
    if hit is not None and hit[0] is terms_obj and hit[1] == obs.num_qubits:
        return hit[2]
    table = _lower_terms(obs)
    for a in table:
        a.setflags(write=False)
    if isinstance(terms_obj, tuple):
        if len(_TERMS_CACHE) > 64:
            _TERMS_CACHE.clear()
        _TERMS_CACHE[id(terms_obj)] = (terms_obj, obs.num_qubits, table)
    return table


class Problem:
    """Owns the numpy tables and the svg_problem that points into them."""

    def __init__(self, circuit, params, obs, input_state, real_sums: bool = False, forward_only: bool = False):
        self.gates, self.derivs = bind(circuit, params, forward_only)
        self.terms, self.products, self.factors = lower_terms(obs)
        self.num_derivs = len(self.derivs)
        basis = basis_index_of(input_state)
        self.amps = None
        local = isinstance(input_state, ShardSlice)
        if basis is None:
            self.amps = np.ascontiguousarray(input_state.amplitudes, dtype=np.complex128)
        p = N.svg_problem()
        p.num_qubits = circuit.num_qubits
        p.num_params = circuit.num_params
        p.num_gates = len(self.gates)
        p.num_derivs = self.num_derivs
        p.num_terms = len(self.terms)
        p.flags = (FLAG_REAL_SUMS if real_sums else 0) | (FLAG_INPUT_LOCAL if local else 0)
        p.gates = self.gates.ctypes.data
        p.derivs = self.derivs.ctypes.data
        p.terms = self.terms.ctypes.data
        p.num_product_terms = len(self.products)
        p.num_factors = len(self.factors)
        p.product_terms = self.products.ctypes.data
        p.factors = self.factors.ctypes.data
        p.input_basis = 0 if basis is None else basis
        p.input_amps = None if self.amps is None else self.amps.ctypes.data
        self.c = p

    @property
    def h2d_state_bytes(self) -> int:
        return 0 if self.amps is None else self.amps.nbytes
