"""Numpy emulator of the device algorithm over the lowered C-ABI tables (TEST ONLY).

Executes exactly what libsvgb200.so is asked to execute -- the svg_problem
tables built by ``paper_2009_02823_b200.lowering`` and the pass order from
``svg_plan_inspect`` -- with dense numpy ops instead of tiles.  It checks the
host side (binding, generator algebra, planner reordering, sum accumulation
order) on a machine without a GPU; the kernels themselves are checked by the
gpu-marked tests.
"""
from __future__ import annotations

import numpy as np

from paper_2009_02823_b200 import _native
from paper_2009_02823_b200.lowering import Problem


def _pauli_apply(vec, a, b, x, z, ny, ctrl):
    idx = np.arange(vec.size, dtype=np.uint64)
    src = idx ^ np.uint64(x)
    par = np.array([bin(int(v)).count("1") & 1 for v in (src & np.uint64(z))]) if vec.size <= 64 else \
        _popcount_parity(src & np.uint64(z))
    ph = (1j ** ny) * np.where(par == 1, -1.0, 1.0)
    out = a * vec + b * ph * vec[src.astype(np.int64)]
    ok = (idx & np.uint64(ctrl)) == np.uint64(ctrl)
    return np.where(ok, out, vec)


def _popcount_parity(v):
    v = v.copy()
    p = np.zeros(v.shape, dtype=np.uint64)
    while np.any(v):
        p ^= v & np.uint64(1)
        v >>= np.uint64(1)
    return p


def _mat_apply(vec, m, targets, ctrl):
    k = len(targets)
    g = 1 << k
    m = np.asarray(m[: g * g]).reshape(g, g)
    idx = np.arange(vec.size, dtype=np.int64)
    tmask = sum(1 << t for t in targets)
    base = idx[((idx & tmask) == 0) & ((idx & ctrl) == ctrl)]
    offs = [sum(((s >> j) & 1) << t for j, t in enumerate(targets)) for s in range(g)]
    groups = np.stack([base + o for o in offs])
    out = vec.copy()
    out[groups] = m @ vec[groups]
    return out


def _apply(vec, gate, field, ctrl_only=True):
    c = gate[field]
    ctrl = int(gate["ctrl_mask"])
    if gate["form"] == _native.FORM_PAULI:
        return _pauli_apply(vec, c[0], c[1], int(gate["x_mask"]), int(gate["z_mask"]), int(gate["n_y"]), ctrl)
    targets = list(gate["targets"][: gate["ntargets"]])
    return _mat_apply(vec, c, targets, ctrl)


def _generator(vec, gate, kvec):
    """K phi restricted to the control subspace (zero elsewhere)."""
    ctrl = int(gate["ctrl_mask"])
    if gate["form"] == _native.FORM_PAULI:
        out = _pauli_apply(vec, kvec[0], kvec[1], int(gate["x_mask"]), int(gate["z_mask"]), int(gate["n_y"]), 0)
    else:
        out = _mat_apply(vec, kvec, list(gate["targets"][: gate["ntargets"]]), 0)
    idx = np.arange(vec.size, dtype=np.int64)
    return np.where((idx & ctrl) == ctrl, out, 0)


def emulate(circuit, params, obs, input_state, tile_qubits=0, sms=0):
    """(sums complex[P], energy, pass_count) computed from the lowered tables."""
    prob = Problem(circuit, np.asarray(params, dtype=float), obs, input_state)
    n = circuit.num_qubits
    order, start, qmasks, k = _native.plan_inspect(prob.c, tile_qubits, sms)
    gates, derivs, terms = prob.gates, prob.derivs, prob.terms
    psi = np.array(input_state.amplitudes, dtype=complex)
    for gi in order:
        psi = _apply(psi, gates[gi], "fwd")
    lam = np.zeros_like(psi)
    for t in terms:
        lam += _pauli_apply(psi, 0.0, t["coeff"], int(t["x_mask"]), int(t["z_mask"]), int(t["n_y"]), 0)
    energy = np.vdot(psi, lam)
    first = np.concatenate([[0], np.cumsum(gates["nderiv"])]).astype(int)
    contrib = np.zeros(len(derivs), dtype=complex)
    for p in range(len(start) - 2, -1, -1):
        for gi in order[start[p]: start[p + 1]][::-1]:
            g = gates[gi]
            for j in range(int(g["nderiv"])):  # generators in the post-gate basis see phi_{i+1}
                d = first[gi] + j
                if derivs[d]["basis"] == 1:
                    contrib[d] = np.vdot(lam, _generator(psi, g, derivs[d]["k"]))
            psi = _apply(psi, g, "rewind")
            for j in range(int(g["nderiv"])):
                d = first[gi] + j
                if derivs[d]["basis"] == 0:
                    contrib[d] = np.vdot(lam, _generator(psi, g, derivs[d]["k"]))
            if gi > 0:
                lam = _apply(lam, g, "adjoint")
    sums = np.zeros(circuit.num_params, dtype=complex)
    for gi in range(len(gates) - 1, -1, -1):
        for j in range(int(gates[gi]["nderiv"])):
            d = first[gi] + j
            sums[derivs[d]["param_ref"]] += contrib[d]
    return sums, complex(energy), (order, start, qmasks, k)
