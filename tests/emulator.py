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


def _pauli_apply(vec, a, b, x, z, ny, ctrl, rank_bits=0, src_vec=None, src_bits=None):
    """a vec + b P vec on a (shard of a) state.  Signs and controls use the
    physical index (local index | rank_bits); ``src_vec``/``src_bits`` supply the
    partner shard when the Pauli flips rank bits (observable terms)."""
    idx = np.arange(vec.size, dtype=np.uint64)
    src = idx ^ np.uint64(x & (vec.size - 1))
    sbits = np.uint64(rank_bits if src_bits is None else src_bits)
    par = _popcount_parity((src | sbits) & np.uint64(z))
    ph = (1j ** ny) * np.where(par == 1, -1.0, 1.0)
    source = vec if src_vec is None else src_vec
    out = a * vec + b * ph * source[src.astype(np.int64)]
    ok = ((idx | np.uint64(rank_bits)) & np.uint64(ctrl)) == np.uint64(ctrl)
    return np.where(ok, out, vec)


def _popcount_parity(v):
    v = v.copy()
    p = np.zeros(v.shape, dtype=np.uint64)
    while np.any(v):
        p ^= v & np.uint64(1)
        v >>= np.uint64(1)
    return p


def _mat_apply(vec, m, targets, ctrl, rank_bits=0):
    k = len(targets)
    g = 1 << k
    m = np.asarray(m[: g * g]).reshape(g, g)
    idx = np.arange(vec.size, dtype=np.int64)
    tmask = sum(1 << t for t in targets)
    base = idx[((idx & tmask) == 0) & (((idx | rank_bits) & ctrl) == ctrl)]
    offs = [sum(((s >> j) & 1) << t for j, t in enumerate(targets)) for s in range(g)]
    groups = np.stack([base + o for o in offs])
    out = vec.copy()
    out[groups] = m @ vec[groups]
    return out


def _apply(vec, gate, field, rank_bits=0):
    c = gate[field]
    ctrl = int(gate["ctrl_mask"])
    if gate["form"] == _native.FORM_PAULI:
        return _pauli_apply(vec, c[0], c[1], int(gate["x_mask"]), int(gate["z_mask"]), int(gate["n_y"]), ctrl,
                            rank_bits)
    targets = list(gate["targets"][: gate["ntargets"]])
    return _mat_apply(vec, c, targets, ctrl, rank_bits)


def _generator(vec, gate, kvec, rank_bits=0):
    """K phi restricted to the control subspace (zero elsewhere)."""
    ctrl = int(gate["ctrl_mask"])
    if gate["form"] == _native.FORM_PAULI:
        out = _pauli_apply(vec, kvec[0], kvec[1], int(gate["x_mask"]), int(gate["z_mask"]), int(gate["n_y"]), 0,
                           rank_bits)
    else:
        out = _mat_apply(vec, kvec, list(gate["targets"][: gate["ntargets"]]), 0, rank_bits)
    idx = np.arange(vec.size, dtype=np.int64)
    return np.where(((idx | rank_bits) & ctrl) == ctrl, out, 0)


def _rank_pauli_parts(m, bit):
    """2x2 factor on a rank bit in the Pauli basis: [(x, z, weight incl. i^n_y)] (engine.cu lowering)."""
    m = np.asarray(m).reshape(2, 2)
    a, d = (m[0, 0] + m[1, 1]) / 2, (m[0, 0] - m[1, 1]) / 2
    b, c = (m[0, 1] + m[1, 0]) / 2, 1j * (m[0, 1] - m[1, 0]) / 2
    return [(0, 0, a), (bit, 0, b), (bit, bit, c * 1j), (0, bit, d)]


def _product_terms(prob, psi, l2p=None, nloc=None, rank=0, fetch=None):
    """sum_t c_t (x)F_t psi over the problem's product terms (dense factor-by-factor
    application; rank-bit factors in Pauli form with partner shards from ``fetch``)."""
    out = np.zeros_like(psi)
    nloc = nloc if nloc is not None else int(np.log2(psi.size))
    for pt in prob.products:
        facs = prob.factors[int(pt["first_factor"]): int(pt["first_factor"]) + int(pt["num_factors"])]
        loc, subs = [], [(0, 0, 1.0 + 0j)]
        for f in facs:
            q = int(f["qubit"]) if l2p is None else l2p[int(f["qubit"])]
            if q < nloc:
                loc.append((q, f["m"]))
                continue
            subs = [(x | x2, z | z2, w * w2) for x, z, w in subs for x2, z2, w2 in _rank_pauli_parts(f["m"], 1 << q)
                    if w * w2 != 0]
        for x, z, w in subs:
            src = psi if x == 0 else fetch(x)
            v = src.copy()
            for q, m in loc:
                v = _mat_apply(v, m, [q], 0)
            src_rank = (rank << nloc) ^ x
            sign = -1.0 if bin(src_rank & z).count("1") & 1 else 1.0
            out += complex(pt["coeff"]) * w * sign * v
    return out


def emulate(circuit, params, obs, input_state, tile_qubits=0, sms=0):
    """(sums complex[P], energy, pass_count) computed from the lowered tables."""
    prob = Problem(circuit, np.asarray(params, dtype=float), obs, input_state)
    order, start, qmasks, k = _native.plan_inspect(prob.c, tile_qubits, sms)
    sums, energy = emulate_order(circuit, params, obs, input_state, order)
    return sums, energy, (order, start, qmasks, k)


def emulate_order(circuit, params, obs, input_state, order):
    """(sums complex[P], energy) of the adjoint sweep with the gates applied in
    `order` (forward) and its reverse (the engine's schedule, dense numpy)."""
    prob = Problem(circuit, np.asarray(params, dtype=float), obs, input_state)
    gates, derivs, terms = prob.gates, prob.derivs, prob.terms
    psi = np.array(input_state.amplitudes, dtype=complex)
    for gi in order:
        psi = _apply(psi, gates[gi], "fwd")
    lam = np.zeros_like(psi)
    for t in terms:
        lam += _pauli_apply(psi, 0.0, t["coeff"], int(t["x_mask"]), int(t["z_mask"]), int(t["n_y"]), 0)
    lam += _product_terms(prob, psi)
    energy = np.vdot(psi, lam)
    first = np.concatenate([[0], np.cumsum(gates["nderiv"])]).astype(int)
    contrib = np.zeros(len(derivs), dtype=complex)
    for gi in list(order)[::-1]:
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
    return sums, complex(energy)


# ---- sharded schedule (one rank's view) -------------------------------------------

def _remap(mask, l2p):
    out = 0
    q = 0
    while mask:
        if mask & 1:
            out |= 1 << l2p[q]
        mask >>= 1
        q += 1
    return out


def _physical(gate, l2p):
    g = gate.copy()
    nt = int(g["ntargets"])
    for j in range(nt):
        g["targets"][j] = l2p[int(gate["targets"][j])]
    for f in ("ctrl_mask", "x_mask", "z_mask"):
        g[f] = _remap(int(gate[f]), l2p)
    return g


def emulate_sharded(circuit, params, obs, input_state, world, rank, exchange, tile_qubits=0, sms=0):
    """One rank's part of the sharded adjoint sweep (the engine's algorithm, dense numpy).

    ``exchange(array, partner) -> array`` swaps equal-size arrays with rank
    ``partner`` (gloo send/recv in the multi-process test).  Returns this
    rank's (per-derivative contributions, energy contribution, schedule).
    """
    prob = Problem(circuit, np.asarray(params, dtype=float), obs, input_state)
    n = circuit.num_qubits
    g = world.bit_length() - 1
    nloc = n - g
    steps, _ = _native.plan_schedule(prob.c, world, tile_qubits, sms)
    gates, derivs, terms = prob.gates, prob.derivs, prob.terms
    rank_bits = rank << nloc
    full = np.array(input_state.amplitudes, dtype=complex)
    psi = full[rank << nloc: (rank + 1) << nloc].copy()

    def swap(buf, gbit, lpos):
        a = (rank >> gbit) & 1
        idx = np.arange(buf.size)
        half = ((idx >> lpos) & 1) == 1 - a
        out = buf.copy()
        out[half] = exchange(np.ascontiguousarray(buf[half]), rank ^ (1 << gbit))
        return out

    l2p = list(range(n))
    maps = []
    for st in steps:  # forward
        maps.append(list(l2p))
        if st[0] == "swap":
            _, gbit, lpos = st
            psi = swap(psi, gbit, lpos)
            pg = nloc + gbit
            la, lb = l2p.index(pg), l2p.index(lpos)
            l2p[la], l2p[lb] = lpos, pg
        else:
            for gi in st[1]:
                psi = _apply(psi, _physical(gates[gi], l2p), "fwd", rank_bits)
    lam = np.zeros_like(psi)
    loc = (1 << nloc) - 1
    fetched = {}
    for t in terms:
        x, z = _remap(int(t["x_mask"]), l2p), _remap(int(t["z_mask"]), l2p)
        xg = x & ~loc
        src = psi
        if xg:
            if xg not in fetched:
                fetched[xg] = exchange(psi, rank ^ (xg >> nloc))
            src = fetched[xg]
        lam += _pauli_apply(psi, 0.0, t["coeff"], x & loc, z, int(t["n_y"]), 0, rank_bits, src, rank_bits ^ xg)

    def fetch(xg):
        if xg not in fetched:
            fetched[xg] = exchange(psi, rank ^ (xg >> nloc))
        return fetched[xg]

    lam += _product_terms(prob, psi, l2p, nloc, rank, fetch)
    energy = np.vdot(psi, lam)
    first = np.concatenate([[0], np.cumsum(gates["nderiv"])]).astype(int)
    contrib = np.zeros(len(derivs), dtype=complex)
    for st, m in zip(steps[::-1], maps[::-1]):  # reverse
        if st[0] == "swap":
            _, gbit, lpos = st
            psi, lam = swap(psi, gbit, lpos), swap(lam, gbit, lpos)
            continue
        for gi in st[1][::-1]:
            gp = _physical(gates[gi], m)
            for j in range(int(gp["nderiv"])):
                d = first[gi] + j
                if derivs[d]["basis"] == 1:
                    contrib[d] = np.vdot(lam, _generator(psi, gp, derivs[d]["k"], rank_bits))
            psi = _apply(psi, gp, "rewind", rank_bits)
            for j in range(int(gp["nderiv"])):
                d = first[gi] + j
                if derivs[d]["basis"] == 0:
                    contrib[d] = np.vdot(lam, _generator(psi, gp, derivs[d]["k"], rank_bits))
            lam = _apply(lam, gp, "adjoint", rank_bits)
    return contrib, complex(energy), steps


def combine(circuit, prob_derivs, contrib):
    """Per-derivative contributions -> sums[P] in the reference's accumulation order."""
    first = np.concatenate([[0], np.cumsum([len(g.param_refs) for g in circuit.gates])]).astype(int)
    sums = np.zeros(circuit.num_params, dtype=complex)
    for gi in range(len(circuit.gates) - 1, -1, -1):
        for j in range(len(circuit.gates[gi].param_refs)):
            sums[circuit.gates[gi].param_refs[j]] += contrib[first[gi] + j]
    return sums
