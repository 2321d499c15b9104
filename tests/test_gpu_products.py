"""GPU parity of product-term observables (letters H, +, - kept as 2x2 factors).

The reference applies an observable term factor by factor
(svgrad/observable.py:79-100); its benchmark operator ``hadamard_all``
(svgrad/observable.py:128-137, svgrad/bench.py:94) is one term of N
Hadamards, 2^N Pauli strings if expanded.  Terms with more than
operators.MAX_EXPANDED_LETTERS such letters run as product-term passes
(k_prod_pass: Walsh-Hadamard butterflies over tiles); these tests pin them
to the oracle on single and sharded engines (rank-bit factors in Pauli form).
"""
import numpy as np
import pytest

import paper_2009_02823_b200 as sv
from conftest import load_golden, max_err

from oracle import oracle

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-10
ENERGY_TOL = 1e-12


def _workload(cfg, n, obs):
    w = sv.build_workload(cfg, n)
    return w.circuit, w.theta, obs


def _engine(shards):
    if shards == 1:
        return None
    eng = sv.distributed.virtual_engine(shards)
    eng.set_option("emulate_transport", 1)
    return eng


@pytest.mark.parametrize("shards", [1, 2, 8])
@pytest.mark.parametrize("cfg,n", [(4, 20), (3, 16)])
def test_hadamard_all_matches_oracle(cfg, n, shards):
    circ, theta, _ = _workload(cfg, n, None)
    obs = sv.builtin_observable("hadamard_all", n)
    eng = _engine(shards)
    stats = {}
    rep = sv.reverse_mode_gradient(circ, theta, obs, sv.BasisState(n), engine=eng, stats=stats)
    vals, energy, counters = oracle.reverse_mode_values(circ, theta, obs, sv.init_basis_state(n).amplitudes)
    assert max_err(rep.values, vals) <= GRAD_TOL
    assert abs(rep.energy - energy) <= ENERGY_TOL
    assert vars(rep.counters) == counters
    assert stats["obs_passes"] >= 2  # n > tile width: a multi-pass product pipeline


@pytest.mark.parametrize("shards", [1, 4])
def test_mixed_product_and_pauli_terms_non_hermitian(shards):
    """Raising / lowering / Hadamard products next to Pauli strings (some letters on the
    rank bits of the sharded engine): the non-Hermitian gradient (two sweeps)."""
    n = 14
    circ, theta, _ = _workload(5, n, None)
    rng = np.random.default_rng(7)
    letters = "IXYZH+-"
    terms = [(0.7, "H+-ZHXH" + "I" * (n - 7)), (0.3 - 0.2j, "I" * (n - 6) + "+H-H+Y"),
             (1.1, "".join(rng.choice(list(letters), n))), (-0.4, "ZZ" + "I" * (n - 2)),
             (0.25j, "H" * n)]
    obs = sv.Observable(n, tuple(terms))
    rep = sv.non_hermitian_gradient(circ, theta, obs, sv.BasisState(n), engine=_engine(shards))
    vals, energy, _ = oracle.non_hermitian_values(circ, theta, obs, sv.init_basis_state(n).amplitudes)
    assert max_err(rep.values, vals) <= GRAD_TOL
    assert abs(rep.energy - energy) <= ENERGY_TOL


def test_expectation_with_product_terms():
    n = 18
    circ, theta, _ = _workload(2, n, None)
    obs = sv.Observable(n, ((0.5, "H" * n), (1.0, "X" + "I" * (n - 1)), (0.2, "HHHH+-+-" + "I" * (n - 8))))
    e = sv.circuit_expectation(circ, theta, obs, sv.BasisState(n))
    assert abs(e - oracle.expectation(circ, theta, obs, sv.init_basis_state(n).amplitudes)) <= ENERGY_TOL


@pytest.mark.slow
def test_hadamard_all_n26_vs_oracle_fixture():
    """hadamard_all at n = 26 (one product term of 26 Hadamards, 2^26 Pauli strings if
    expanded) against the oracle fixture (tests/golden/make_oracle_n30.py hadamard_n26)."""
    from golden.make_oracle_n30 import workload

    gold = load_golden("oracle_hadamard_n26.json")["hadamard_n26"]
    w = workload("hadamard_n26")
    rep = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, sv.BasisState(w.num_qubits))
    assert max_err(rep.values, np.asarray(gold["values_real"], dtype=complex)) <= GRAD_TOL
    assert abs(rep.energy - complex(*gold["energy"])) <= ENERGY_TOL
    assert vars(rep.counters) == gold["counters"]
