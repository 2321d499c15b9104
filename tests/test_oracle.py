"""Pin the CPU oracle (oracle/) against the reference's own outputs.

tests/golden/*.json were produced by running the REFERENCE implementation
(tests/golden/make_golden.py); the oracle restatement must reproduce every
value, energy and exact op count before it is trusted as the checker for
the GPU path and for sizes the reference cannot run.
"""
import numpy as np
import pytest

from cases import config_cases, small_cases
from conftest import cvec, load_golden, materialize, max_err

from oracle import oracle

GOLD = load_golden()
CASES = {**small_cases(), **config_cases()}


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_golden(name):
    rec = GOLD[name]
    circ, theta, obs, inp, method = materialize(CASES[name])
    assert circ.num_params == rec["num_params"] and len(circ.gates) == rec["num_gates"]
    assert np.sum(theta) == pytest.approx(rec["theta_sum"], abs=0)
    if method == "non_hermitian":
        values, energy, counters = oracle.non_hermitian_values(circ, theta, obs, inp.amplitudes)
    else:
        values, energy, counters = oracle.reverse_mode_values(circ, theta, obs, inp.amplitudes)
    assert max_err(values, cvec(rec["values"])) <= 1e-12
    assert abs(energy - complex(*rec["energy"])) <= 1e-12
    assert counters == rec["counters"]


def test_oracle_against_reference_gradient_engine():
    """Second pin: the reference's O(P^2) engine agrees with the oracle too."""
    for name in ("family_C4_0", "all_kinds_6_random", "cfg1"):
        rec = GOLD[name]
        circ, theta, obs, inp, _ = materialize(CASES[name])
        values, _, _ = oracle.reverse_mode_values(circ, theta, obs, inp.amplitudes)
        assert max_err(values, cvec(rec["reference_gradient_values"])) <= 1e-10


def test_oracle_negative_control():
    """A 1% perturbation of the derivative scalars must be caught by the same check."""
    circ, theta, obs, inp, _ = materialize(CASES["family_D4_0"])
    good = oracle.sweep(circ, theta, obs, inp.amplitudes)
    bad = oracle.sweep(circ, theta, obs, inp.amplitudes, deriv_scale=1.01)
    assert max_err(2 * bad.sums.real, 2 * good.sums.real) > 1e-4


def test_oracle_thread_count_invariance():
    circ, theta, obs, inp, _ = materialize(CASES["cfg2_n12"])
    one = oracle.sweep(circ, theta, obs, inp.amplitudes, threads=1)
    many = oracle.sweep(circ, theta, obs, inp.amplitudes, threads=4)
    assert max_err(many.sums, one.sums) <= 1e-12


@pytest.mark.parametrize("name", sorted(n for n in CASES if GOLD[n]["method"] == "reverse"))
def test_lean_sweep_matches_reference_golden(name):
    """oracle_sweep_lean (the n = 30 fixture generator: probe contracted group by
    group, basis-index input) against the reference's own outputs."""
    rec = GOLD[name]
    circ, theta, obs, inp, _ = materialize(CASES[name])
    r = oracle.sweep_lean(circ, theta, obs, inp.amplitudes)
    assert max_err(2.0 * r.sums.real, cvec(rec["values"])) <= 1e-12
    assert abs(r.energy - complex(*rec["energy"])) <= 1e-12
    assert r.counters == rec["counters"]


@pytest.mark.parametrize("cfg,n", [(4, 16), (5, 15), (3, 14), (2, 14)])
def test_lean_sweep_matches_literal_with_basis_input(cfg, n):
    import paper_2009_02823_b200 as sv

    w = sv.build_workload(cfg, n)
    a = oracle.sweep(w.circuit, w.theta, w.observable, sv.init_basis_state(n).amplitudes)
    b = oracle.sweep_lean(w.circuit, w.theta, w.observable, None, 0)
    assert max_err(b.sums, a.sums) <= 1e-13
    assert abs(a.energy - b.energy) <= 1e-13
    assert a.counters == b.counters


def test_op_count_model_matches_counters():
    """oracle.op_counts (bench.py's CPU-baseline model) counts the same schedule the
    counters report: gate applies = 3G-1 plus the derivative/observable applies."""
    import paper_2009_02823_b200 as sv

    w = sv.build_workload(4, 8)
    c = oracle.op_counts(w.circuit, w.observable)
    G, A = w.num_gates, w.circuit.num_params
    factors = sum(sum(ch != "I" for ch in f) for _, f in w.observable.terms)
    assert c["apply_1q"] + c["apply_1q_ctrl"] + c["apply_2q"] == (3 * G - 1) + 2 * A + factors
    assert c["clone"] == A + 2 + len(w.observable.terms)
    assert c["inner"] == A + 1


def test_n30_fixtures_are_pinned_to_this_oracle():
    """The committed n = 30 fixtures (tests/golden/make_oracle_n30.py) match the
    workload generator and the oracle source they were produced from."""
    import hashlib
    import json
    import os

    from golden.digest import circuit_digest, obs_digest

    here = os.path.join(os.path.dirname(__file__), "golden")
    found = 0
    from golden.make_oracle_n30 import CASES, workload

    for name in CASES:
        path = os.path.join(here, f"oracle_{name}.json")
        if not os.path.exists(path):
            continue
        found += 1
        rec = json.load(open(path))["cases"][name]
        w = workload(name)
        assert rec["circuit_digest"] == circuit_digest(w.circuit)
        assert rec["obs_digest"] == obs_digest(w.observable)
        assert rec["theta_sum"] == pytest.approx(float(np.sum(w.theta)), abs=0)
        assert len(rec["values_real"]) == w.circuit.num_params
        G, A = w.num_gates, w.circuit.num_params
        assert rec["counters"] == {"gate_applies": 3 * G - 1, "derivative_applies": A, "clones": A + 2,
                                   "inner_products": A, "observable_applies": 1}
        assert rec["sums_imag_max"] >= 0.0
        with open(oracle.SRC, "rb") as f:
            src = hashlib.sha256(f.read()).hexdigest()
        assert rec["oracle_sha256"] == src, "oracle source changed since the fixture was generated"
    if not found:
        pytest.skip("no n = 30 fixtures generated yet")
