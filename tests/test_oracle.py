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
