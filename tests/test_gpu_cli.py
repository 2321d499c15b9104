"""CLI and finite-difference gradient on the GPU:
the `grad` front end's report against the reference CLI's own output for the
same files (tests/golden/golden_textio.json), and central differences through
the GPU expectation path against the fused reverse sweep."""
import json
import os

import numpy as np
import pytest

import paper_2009_02823_b200 as sv
from paper_2009_02823_b200 import cli
from cases import config_cases
from conftest import cvec, load_golden, materialize, max_err

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden_textio.json")))


def _parse_report(text):
    energy, values, counters = None, {}, None
    for line in text.strip().splitlines():
        tok = line.split()
        if tok[0] == "energy":
            energy = complex(float(tok[1]), float(tok[2]))
        elif tok[0] == "counters":
            counters = dict(t.split("=") for t in tok[1:])
        else:
            values[tok[0]] = complex(float(tok[1]), float(tok[2]))
    return energy, values, counters


@pytest.mark.parametrize("i", range(len(GOLD["cli"])))
def test_cli_grad_matches_reference_cli(i, tmp_path, capsys):
    rec = GOLD["cli"][i]
    circ = tmp_path / "c.circ"
    circ.write_text(rec["circuit"])
    obs = rec["observable"]
    if obs.startswith("obs:"):
        (tmp_path / "o.obs").write_text(obs[4:])
        obs = str(tmp_path / "o.obs")
    code = cli.main(["grad", str(circ), obs, rec["params"], "--method", rec["method"]])
    assert code == rec["exit_code"]
    if code != 0:
        return
    out = capsys.readouterr().out
    e, vals, counters = _parse_report(out)
    e_ref, vals_ref, counters_ref = _parse_report(rec["stdout"])
    assert vals.keys() == vals_ref.keys() and counters == counters_ref
    assert abs(e - e_ref) <= 1e-12
    for k in vals:
        assert abs(vals[k] - vals_ref[k]) <= 1e-10 * max(1.0, abs(vals_ref[k]))
    for line in out.splitlines():  # full-precision rendering (17 significant digits)
        if line.startswith("p0 "):
            tok = line.split()[1]
            assert tok == f"{float(tok):.17g}"


def test_cli_output_file_and_unwritable(tmp_path):
    circ = tmp_path / "ry.circ"
    circ.write_text("qubits 1\nparams 1\nry q0 p0\n")
    dest = tmp_path / "out.txt"
    assert cli.main(["grad", str(circ), "z_all", "0.7", "-o", str(dest)]) == 0
    _, vals, _ = _parse_report(dest.read_text())
    assert abs(vals["p0"].real + np.sin(0.7)) <= 1e-12
    assert cli.main(["grad", str(circ), "z_all", "0.7", "-o", str(tmp_path / "no" / "dir" / "x")]) == cli.EXIT_OUTPUT


@pytest.mark.parametrize("name", ["cfg1", "cfg3_n14", "cfg5_n15"])
def test_finite_difference_matches_reverse(name):
    """Reference tolerance between FD (delta 1e-5) and the adjoint: 1e-6 (pkg/tests/test_gradients.py)."""
    rec = load_golden()[name]
    circ, theta, obs, inp, _ = materialize(config_cases()[name])
    fd = sv.finite_difference_gradient(circ, theta, obs, inp)
    assert max_err(fd.values, cvec(rec["values"])) <= 1e-6
    assert abs(fd.energy - complex(*rec["energy"])) <= 1e-12
    assert fd.counters.observable_applies == 2 * circ.num_params + 1


def test_cli_fd_method(tmp_path, capsys):
    circ = tmp_path / "ry.circ"
    circ.write_text("qubits 2\nparams 2\nry q0 p0\ncx q0 q1\nrx q1 p1\n")
    assert cli.main(["grad", str(circ), "hadamard_all", "0.4,1.3", "--method", "fd"]) == 0
    _, fd, _ = _parse_report(capsys.readouterr().out)
    assert cli.main(["grad", str(circ), "hadamard_all", "0.4,1.3"]) == 0
    _, rev, _ = _parse_report(capsys.readouterr().out)
    for k in rev:
        assert abs(fd[k] - rev[k]) <= 1e-6


def test_reverse_mode_time_is_linear_in_parameters():
    """The paper's scaling claim as the reference's acceptance criterion 3 states it
    for reverse mode (log-log slope of time vs P in [0.75, 1.35]; reference
    pkg/tests/test_acceptance.py:97-117), here on the GPU at n = 20, P = 320..2560."""
    import time

    n = 20
    obs = sv.Observable(n, tuple((1.0, "I" * i + "ZZ" + "I" * (n - i - 2)) for i in range(n - 1)))
    inp = sv.BasisState(n)
    ps, ts = [], []
    for L in (8, 16, 32, 64):
        gates, p = [], 0
        for _ in range(L):
            for q in range(n):
                gates.append(sv.ry(q, p))
                p += 1
            for q in range(n):
                gates.append(sv.rz(q, p))
                p += 1
            gates += [sv.cx(q, q + 1) for q in range(n - 1)]
        circ = sv.Circuit(n, tuple(gates), p)
        theta = np.random.default_rng([L]).uniform(0, 2 * np.pi, p)
        sv.reverse_mode_gradient(circ, theta, obs, inp)  # compile / warm up
        best = float("inf")
        for _ in range(5):
            t0 = time.perf_counter()
            sv.reverse_mode_gradient(circ, theta, obs, inp)
            best = min(best, time.perf_counter() - t0)
        ps.append(p)
        ts.append(best)
    slope = np.polyfit(np.log(ps), np.log(ts), 1)[0]
    assert 0.75 <= slope <= 1.35, (slope, ts)


@pytest.mark.parametrize("name", ["single_ry_3", "family_A4_1", "family_D5_0", "repeated_rz", "unreferenced_slot",
                                  "no_params", "multi_param_fd", "shared_slot", "non_unitary", "all_kinds_4_random",
                                  "all_kinds_6_basis", "random_input_family_C", "cfg1"])
def test_reference_gradient_quadratic_schedule(name):
    """The reference's O(P^2) schedule on the GPU (svgrad/gradients.py:201-237, one
    derivative-inserted forward sweep per parameter occurrence) against the reference's
    reverse-mode outputs (the reference pins reverse == reference to 1e-11,
    pkg/tests/test_gradients.py:131-144), with the quadratic counters
    (pkg/tests/test_gradients.py:324-333)."""
    from cases import small_cases

    rec = load_golden()[name]
    circ, theta, obs, inp, _ = materialize({**small_cases(), **config_cases()}[name])
    rep = sv.reference_gradient(circ, theta, obs, inp)
    assert max_err(rep.values, cvec(rec["values"])) <= 1e-10
    assert abs(rep.energy - complex(*rec["energy"])) <= 1e-12
    G = len(circ.gates)
    A = sum(len(g.param_refs) for g in circ.gates)
    assert vars(rep.counters) == {"gate_applies": G + A * (G - 1), "derivative_applies": A, "clones": A + 1,
                                  "inner_products": A, "observable_applies": 1}


def test_reference_gradient_rejects_non_hermitian():
    circ = sv.Circuit(1, (sv.ry(0, 0),), 1)
    obs = sv.Observable(1, ((1.0, "+"),))
    with pytest.raises(ValueError, match="non_hermitian_gradient"):
        sv.reference_gradient(circ, [0.1], obs, sv.init_basis_state(1))
