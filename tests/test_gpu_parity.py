"""GPU parity: the CUDA path through the drop-in API vs the reference's golden outputs and the oracle.

Bar (BASELINE.json north_star): every gradient entry within 1e-10 abs-or-rel,
energy within 1e-12; exact OpCounters.  Everything here runs through
``paper_2009_02823_b200.reverse_mode_gradient`` -> libsvgb200.so (C-ABI).
"""
import numpy as np
import pytest

import paper_2009_02823_b200 as sv
from cases import config_cases, large_config_cases, small_cases
from conftest import cvec, load_golden, materialize, max_err

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-10
ENERGY_TOL = 1e-12

GOLD = load_golden()
SMALL = {**small_cases(), **config_cases()}


def _run(circ, theta, obs, inp, method):
    if method == "non_hermitian":
        return sv.non_hermitian_gradient(circ, theta, obs, inp)
    return sv.reverse_mode_gradient(circ, theta, obs, inp)


@pytest.mark.parametrize("name", sorted(SMALL))
def test_gpu_matches_reference_golden(name):
    rec = GOLD[name]
    circ, theta, obs, inp, method = materialize(SMALL[name])
    rep = _run(circ, theta, obs, inp, method)
    assert max_err(rep.values, cvec(rec["values"])) <= GRAD_TOL
    assert abs(rep.energy - complex(*rec["energy"])) <= ENERGY_TOL
    assert vars(rep.counters) == rec["counters"]
    if method == "reverse":
        assert np.all(rep.values.imag == 0.0)


@pytest.mark.parametrize("name", ["cfg2", "cfg3_n20", "cfg4_n20", "cfg5_n20", "cfg3"])
def test_gpu_matches_reference_golden_large(name):
    gold = load_golden(f"golden_{name}.json")[name]
    circ, theta, obs, inp, method = materialize(large_config_cases()[name])
    rep = _run(circ, theta, obs, inp, method)
    err = max_err(rep.values, cvec(gold["values"]))
    assert err <= GRAD_TOL, err
    assert abs(rep.energy - complex(*gold["energy"])) <= ENERGY_TOL
    assert vars(rep.counters) == gold["counters"]


_VARIANTS = {  # generated-kernel plan options (engine defaults: auto)
    "wide_tiles": {"tile_qubits": 12, "tile_fwd": -1},
    "fwd_split_13": {"tile_qubits": 12, "tile_fwd": 13},
    "fwd_split_12": {"tile_qubits": 11, "tile_fwd": 12},
    "low_qubits_5": {"low_qubits": 5},
    "low_qubits_4_wide": {"low_qubits": 4, "tile_qubits": 12},
    "reg_bits_3": {"reg_bits": 3},
    "low_qubits_3": {"low_qubits": 3},
}


@pytest.mark.parametrize("variant", sorted(_VARIANTS))
@pytest.mark.parametrize("name", ["cfg3_n20", "cfg5_n20"])
def test_generated_kernel_variants_match_reference_golden(name, variant):
    """Every plan option of the generated kernels (tile widths, separate forward
    schedules, forced low qubits, register bits) against the golden."""
    gold = load_golden(f"golden_{name}.json")[name]
    circ, theta, obs, inp, method = materialize(large_config_cases()[name])
    opts = {"jit": 2, **_VARIANTS[variant]}
    eng = sv._native.engine()
    try:
        for k, v in opts.items():
            eng.set_option(k, v)
        rep = _run(circ, theta, obs, inp, method)
    finally:
        for k, v in {"jit": 1, "tile_qubits": 0, "tile_fwd": 0, "low_qubits": 4, "reg_bits": 0}.items():
            eng.set_option(k, v)
    assert max_err(rep.values, cvec(gold["values"])) <= GRAD_TOL
    assert abs(rep.energy - complex(*gold["energy"])) <= ENERGY_TOL


@pytest.mark.parametrize("tile", [0, 7, 8, 9, 11, 12])
def test_tile_size_invariance(tile):
    """Different pass plans (tile widths) reorder commuting gates only."""
    circ, theta, obs, inp, _ = materialize(SMALL["cfg5_n15"])
    eng = sv._native.engine()
    eng.set_option("tile_qubits", tile)
    try:
        rep = sv.reverse_mode_gradient(circ, theta, obs, inp)
    finally:
        eng.set_option("tile_qubits", 0)
    rec = GOLD["cfg5_n15"]
    assert max_err(rep.values, cvec(rec["values"])) <= GRAD_TOL
    assert abs(rep.energy - complex(*rec["energy"])) <= ENERGY_TOL


def _with_options(opts, fn):
    eng = sv._native.engine()
    for k, v in opts.items():
        eng.set_option(k, v)
    try:
        return fn()
    finally:
        for k in opts:
            eng.set_option(k, 0)


@pytest.mark.parametrize("name", ["cfg2_n12", "cfg3_n14", "cfg4_n16", "cfg5_n15", "cfg1"])
@pytest.mark.parametrize("kernel,reg_bits", [(1, 0), (2, 3), (2, 4)])
def test_both_kernel_families_match_golden(name, kernel, reg_bits):
    """Shared-memory tiles (1) and interpreted register tiles (2, R = 3 / 4) against the reference's outputs."""
    rec = GOLD[name]
    circ, theta, obs, inp, _ = materialize(SMALL[name])
    rep = _with_options({"kernel": kernel, "reg_bits": reg_bits},
                        lambda: sv.reverse_mode_gradient(circ, theta, obs, inp))
    assert max_err(rep.values, cvec(rec["values"])) <= GRAD_TOL
    assert abs(rep.energy - complex(*rec["energy"])) <= ENERGY_TOL


@pytest.mark.parametrize("n", [9, 10, 12])
@pytest.mark.parametrize("method", ["reverse", "non_hermitian"])
def test_every_gate_kind_in_register_tiles(n, method):
    """Dense-matrix gates (shared-memory segments), controls, 2-qubit Paulis, repeated
    parameters and complex generators, at sizes that use the register-tile kernels."""
    from cases import all_kinds_circuit, mixed_observable, random_amplitudes
    from oracle import oracle

    circ = all_kinds_circuit(sv, n)
    theta = np.random.default_rng([5, n]).uniform(-np.pi, 2 * np.pi, circ.num_params)
    complex_obs = method == "non_hermitian"
    obs = mixed_observable(sv, n, 21, count=12, letters="XYZ+-" if complex_obs else "XYZH", complex_coeffs=complex_obs)
    inp = sv.StateVector(n, random_amplitudes(n, 9))
    for tile in (0, 9, 10):
        if tile > n:
            continue
        if complex_obs:
            rep = _with_options({"tile_qubits": tile}, lambda: sv.non_hermitian_gradient(circ, theta, obs, inp))
            vals, energy, _ = oracle.non_hermitian_values(circ, theta, obs, inp.amplitudes)
        else:
            rep = _with_options({"tile_qubits": tile}, lambda: sv.reverse_mode_gradient(circ, theta, obs, inp))
            vals, energy, _ = oracle.reverse_mode_values(circ, theta, obs, inp.amplitudes)
        assert max_err(rep.values, vals) <= GRAD_TOL, tile
        assert abs(rep.energy - energy) <= ENERGY_TOL


def test_pass_cap_invariance():
    circ, theta, obs, inp, _ = materialize(SMALL["cfg3_n14"])
    eng = sv._native.engine()
    ref = sv.reverse_mode_gradient(circ, theta, obs, inp)
    eng.set_option("max_gates_per_pass", 3)
    try:
        rep = sv.reverse_mode_gradient(circ, theta, obs, inp)
    finally:
        eng.set_option("max_gates_per_pass", 0)
    assert max_err(rep.values, ref.values) <= 1e-12


def test_bitwise_deterministic():
    circ, theta, obs, inp, _ = materialize(SMALL["cfg4_n16"])
    a = sv.reverse_mode_gradient(circ, theta, obs, inp)
    b = sv.reverse_mode_gradient(circ, theta, obs, inp)
    assert np.array_equal(a.values, b.values) and a.energy == b.energy


def test_basis_fast_path_equals_dense_input():
    circ, theta, obs, _, _ = materialize(SMALL["cfg2_n12"])
    dense = sv.reverse_mode_gradient(circ, theta, obs, sv.init_basis_state(12, 5))
    fast = sv.reverse_mode_gradient(circ, theta, obs, sv.BasisState(12, 5))
    assert max_err(fast.values, dense.values) <= 1e-13


def test_accepts_reference_style_objects_via_duck_typing():
    """Inputs are duck-typed: a foreign Circuit/Observable/StateVector works."""
    from types import SimpleNamespace as NS

    circ, theta, obs, inp, _ = materialize(SMALL["family_B4_0"])
    foreign_gates = tuple(NS(kind=g.kind, targets=g.targets, controls=g.controls, param_refs=g.param_refs)
                          for g in circ.gates)
    fc = NS(num_qubits=circ.num_qubits, gates=foreign_gates, num_params=circ.num_params)
    fo = NS(num_qubits=obs.num_qubits, terms=obs.terms, is_hermitian=True)
    fs = NS(num_qubits=inp.num_qubits, amplitudes=inp.amplitudes)
    rep = sv.reverse_mode_gradient(fc, theta, fo, fs)
    assert max_err(rep.values, cvec(GOLD["family_B4_0"]["values"])) <= GRAD_TOL


def test_errors_match_reference():
    z1 = sv.Observable(1, ((1.0, "Z"),))
    circ = sv.Circuit(1, (sv.ry(0, 0),), 1)
    with pytest.raises(ValueError, match="non_hermitian_gradient"):
        sv.reverse_mode_gradient(circ, [0.1], sv.Observable(1, ((1.0, "+"),)), sv.init_basis_state(1))
    with pytest.raises(ValueError):
        sv.reverse_mode_gradient(circ, [0.1, 0.2], z1, sv.init_basis_state(1))
    with pytest.raises(ValueError):
        sv.reverse_mode_gradient(circ, [0.1], sv.builtin_observable("z_all", 2), sv.init_basis_state(1))
    bad = sv.Gate(sv.NonUnitary(lambda t: np.zeros((2, 2)), 1), (0,), (), (0,))
    with pytest.raises(sv.NonInvertibleGateError, match="gate 1"):
        sv.reverse_mode_gradient(sv.Circuit(1, (sv.ry(0, 0), bad), 1), [0.1], z1, sv.init_basis_state(1))


def test_live_state_audit_peak():
    audit = sv.LiveStateAudit()
    circ = sv.Circuit(2, tuple(sv.rx(i % 2, i) for i in range(10)), 10)
    sv.reverse_mode_gradient(circ, np.zeros(10), sv.builtin_observable("z_all", 2), sv.init_basis_state(2), audit=audit)
    assert audit.peak == 4 and audit.live == 0


def test_negative_control_is_detected():
    circ, theta, obs, inp, _ = materialize(SMALL["family_D4_0"])
    with sv.perturbed_derivative_scale(1.01):
        rep = sv.reverse_mode_gradient(circ, theta, obs, inp)
    assert max_err(rep.values, cvec(GOLD["family_D4_0"]["values"])) > 1e-4


def test_expectation_matches_oracle():
    from oracle import oracle

    circ, theta, obs, inp, _ = materialize(SMALL["all_kinds_6_random"])
    e = sv.circuit_expectation(circ, theta, obs, inp)
    assert abs(e - oracle.expectation(circ, theta, obs, inp.amplitudes)) <= ENERGY_TOL


@pytest.mark.parametrize("n", [11, 13])
def test_wide_flip_terms_use_untiled_pass(n):
    """hadamard_all expands into Pauli strings flipping up to n qubits (> tile width)."""
    from oracle import oracle

    circ = sv.Circuit(n, tuple(sv.ry(q, q) for q in range(n)) + tuple(sv.cx(q, (q + 1) % n) for q in range(n)), n)
    theta = np.linspace(0.1, 2.9, n)
    obs = sv.builtin_observable("hadamard_all", n)
    inp = sv.init_basis_state(n)
    rep = sv.reverse_mode_gradient(circ, theta, obs, inp)
    vals, energy, _ = oracle.reverse_mode_values(circ, theta, obs, inp.amplitudes)
    assert max_err(rep.values, vals) <= GRAD_TOL
    assert abs(rep.energy - energy) <= ENERGY_TOL


@pytest.mark.parametrize("cfg,n", [(3, 22), (5, 21)])
def test_gpu_matches_oracle_midsize(cfg, n):
    """Sizes between the fixtures: the pinned C oracle is the checker."""
    from oracle import oracle

    w = sv.build_workload(cfg, n)
    inp = sv.init_basis_state(n)
    rep = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp)
    vals, energy, counters = oracle.reverse_mode_values(w.circuit, w.theta, w.observable, inp.amplitudes)
    assert max_err(rep.values, vals) <= GRAD_TOL
    assert abs(rep.energy - energy) <= ENERGY_TOL
    assert vars(rep.counters) == counters


def _parameter_shift(w, k):
    """Exact for alpha=-1/2 Pauli rotations: g_k = [E(t+pi/2) - E(t-pi/2)] / 2."""
    inp = sv.BasisState(w.num_qubits)
    tp, tm = w.theta.copy(), w.theta.copy()
    tp[k] += np.pi / 2
    tm[k] -= np.pi / 2
    ep = sv.circuit_expectation(w.circuit, tp, w.observable, inp)
    em = sv.circuit_expectation(w.circuit, tm, w.observable, inp)
    return ((ep - em) / 2).real


@pytest.mark.slow
def test_full_size_cfg4_vs_oracle_fixture():
    """BASELINE cfg 4 at its full size (n = 30, 16 GiB per state) on one engine against
    the full-size oracle fixture (tests/golden/make_oracle_n30.py; the reference itself
    would need ~0.5 TiB): every entry <= 1e-10 abs-or-rel, energy <= 1e-12, counters exact."""
    gold = load_golden("oracle_cfg4.json")["cfg4"]
    w = sv.build_workload(4)
    rep = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, sv.BasisState(w.num_qubits))
    assert max_err(rep.values, np.asarray(gold["values_real"], dtype=complex)) <= GRAD_TOL
    assert abs(rep.energy - complex(*gold["energy"])) <= ENERGY_TOL
    assert vars(rep.counters) == gold["counters"]
    assert np.all(rep.values.imag == 0.0)


@pytest.mark.slow
def test_full_size_cfg3_parameter_shift():
    """cfg 3 at n = 26 (also pinned to the reference's own full-size run above):
    the size-independent parameter-shift identity on three entries, and the
    forward-only expectation path."""
    w = sv.build_workload(3)
    rep = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, sv.BasisState(w.num_qubits))
    for k in (0, w.circuit.num_params // 2, w.circuit.num_params - 1):
        assert abs(rep.values[k].real - _parameter_shift(w, k)) <= GRAD_TOL
    e = sv.circuit_expectation(w.circuit, w.theta, w.observable, sv.BasisState(w.num_qubits))
    assert abs(e - rep.energy) <= ENERGY_TOL


@pytest.mark.parametrize("name", ["cfg2_n12", "cfg3_n14", "cfg4_n16", "cfg5_n15", "cfg1", "family_D9_random",
                                  "all_kinds_6_random", "nh_all_kinds_6"])
@pytest.mark.parametrize("reg_bits", [3, 4])
def test_circuit_specialised_kernels_match_golden(name, reg_bits):
    """jit=2: every register-tile pass runs as a generated, NVRTC-compiled kernel."""
    rec = GOLD[name]
    circ, theta, obs, inp, method = materialize(SMALL[name])
    stats = {}
    run = (lambda: sv.non_hermitian_gradient(circ, theta, obs, inp)) if method == "non_hermitian" else \
        (lambda: sv.reverse_mode_gradient(circ, theta, obs, inp, stats=stats))
    rep = _with_options({"jit": 2, "reg_bits": reg_bits, "tile_qubits": 9}, run)
    sv._native.engine().set_option("jit", 1)
    assert max_err(rep.values, cvec(rec["values"])) <= GRAD_TOL
    assert abs(rep.energy - complex(*rec["energy"])) <= ENERGY_TOL
    if stats and circ.num_qubits >= 10:
        assert stats["jit_passes"] > 0


@pytest.mark.parametrize("n", [10, 12])
@pytest.mark.parametrize("method", ["reverse", "non_hermitian"])
def test_circuit_specialised_every_gate_kind(n, method):
    from cases import all_kinds_circuit, mixed_observable, random_amplitudes
    from oracle import oracle

    circ = all_kinds_circuit(sv, n)
    theta = np.random.default_rng([11, n]).uniform(-np.pi, 2 * np.pi, circ.num_params)
    complex_obs = method == "non_hermitian"
    obs = mixed_observable(sv, n, 5, count=12, letters="XYZ+-" if complex_obs else "XYZH", complex_coeffs=complex_obs)
    inp = sv.StateVector(n, random_amplitudes(n, 3))
    fn = sv.non_hermitian_gradient if complex_obs else sv.reverse_mode_gradient
    rep = _with_options({"jit": 2, "tile_qubits": 9}, lambda: fn(circ, theta, obs, inp))
    sv._native.engine().set_option("jit", 1)
    if complex_obs:
        vals, energy, _ = oracle.non_hermitian_values(circ, theta, obs, inp.amplitudes)
    else:
        vals, energy, _ = oracle.reverse_mode_values(circ, theta, obs, inp.amplitudes)
    assert max_err(rep.values, vals) <= GRAD_TOL
    assert abs(rep.energy - energy) <= ENERGY_TOL


@pytest.mark.parametrize("cfg,n", [(2, 20), (3, 20), (4, 20), (5, 20)])
def test_circuit_specialised_equals_interpreted(cfg, n):
    w = sv.build_workload(cfg, n)
    inp = sv.BasisState(n)
    ref = _with_options({"jit": 0}, lambda: sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp))
    sv._native.engine().set_option("jit", 1)
    stats = {}
    rep = _with_options({"jit": 2}, lambda: sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp,
                                                                     stats=stats))
    sv._native.engine().set_option("jit", 1)
    assert stats["jit_passes"] > 0
    assert max_err(rep.values, ref.values) <= 1e-11
    assert abs(rep.energy - ref.energy) <= ENERGY_TOL


def _random_circuit(n, seed, num_gates=160):
    """Seeded random mix of every register-capable gate shape (rotations on lane /
    register / warp / off-tile qubits, controlled rotations, Pauli-product rotations,
    fixed Paulis, CNOTs) plus a few dense gates, with repeated parameters."""
    rng = np.random.default_rng([seed, n, 99])
    gates, P = [], 24
    for _ in range(num_gates):
        r = rng.random()
        q = [int(x) for x in rng.choice(n, size=3, replace=False)]
        p = int(rng.integers(0, P))
        if r < 0.30:
            gates.append({0: sv.rx, 1: sv.ry, 2: sv.rz}[int(rng.integers(0, 3))](q[0], p))
        elif r < 0.45:
            gates.append({0: sv.crx, 1: sv.cry, 2: sv.crz}[int(rng.integers(0, 3))](q[0], q[1], p))
        elif r < 0.60:
            axes = "".join("XYZ"[int(i)] for i in rng.integers(0, 3, size=2))
            gates.append(sv.rp(axes, (q[0], q[1]), p))
        elif r < 0.72:
            gates.append(sv.cx(q[0], q[1]))
        elif r < 0.84:
            gates.append(sv.fixed("xyz"[int(rng.integers(0, 3))], q[0]))
        elif r < 0.90:
            gates.append(sv.fixed("h", q[0]))
        elif r < 0.95:
            gates.append(sv.phase_gate(q[0], p))
        else:
            gates.append(sv.Gate(sv.PauliRotation("X", alpha=0.75), (q[0],), (q[1], q[2]), (p,)))
    return sv.Circuit(n, tuple(gates), P)


@pytest.mark.parametrize("n,seed", [(18, 1), (19, 2), (20, 3), (24, 4)])
def test_random_circuits_match_oracle(n, seed):
    """Randomised gate mixes at sizes where the generated kernels run with their
    default plans (free-lane layouts, carried scales, fused diagonal runs, literal
    permutation signs; 12-qubit tiles at 24 qubits) against the C oracle."""
    from cases import mixed_observable
    from oracle import oracle

    circ = _random_circuit(n, seed, num_gates=120 if n >= 24 else 160)
    theta = np.random.default_rng([seed, 5]).uniform(-np.pi, 2 * np.pi, circ.num_params)
    obs = mixed_observable(sv, n, seed, count=10)
    inp = sv.init_basis_state(n)
    stats = {}
    rep = sv.reverse_mode_gradient(circ, theta, obs, inp, stats=stats)
    vals, energy, counters = oracle.reverse_mode_values(circ, theta, obs, inp.amplitudes)
    assert stats["jit_passes"] > 0
    assert max_err(rep.values, vals) <= GRAD_TOL
    assert abs(rep.energy - energy) <= ENERGY_TOL
    assert vars(rep.counters) == counters


@pytest.mark.parametrize("shards", [2, 4])
def test_random_circuits_sharded_match_oracle(shards):
    """The same random mixes split over virtual shards (qubit swaps, rank-bit signs
    and controls, partner fetches) with the generated kernels (>= 12 local qubits)."""
    from cases import mixed_observable, random_amplitudes
    from oracle import oracle

    n = 20
    circ = _random_circuit(n, 10 + shards)
    theta = np.random.default_rng([shards, 6]).uniform(-np.pi, 2 * np.pi, circ.num_params)
    obs = mixed_observable(sv, n, shards, count=10)
    inp = sv.StateVector(n, random_amplitudes(n, shards))
    eng = sv.distributed.virtual_engine(shards)
    eng.set_option("emulate_transport", 1)
    stats = {}
    rep = sv.reverse_mode_gradient(circ, theta, obs, inp, engine=eng, stats=stats)
    vals, energy, _ = oracle.reverse_mode_values(circ, theta, obs, inp.amplitudes)
    assert stats["jit_passes"] > 0 and stats["swaps"] > 0
    assert max_err(rep.values, vals) <= GRAD_TOL
    assert abs(rep.energy - energy) <= ENERGY_TOL


def test_random_circuit_non_hermitian_matches_oracle():
    from cases import mixed_observable
    from oracle import oracle

    n = 19
    circ = _random_circuit(n, 21)
    theta = np.random.default_rng([21, 7]).uniform(-np.pi, 2 * np.pi, circ.num_params)
    obs = mixed_observable(sv, n, 21, count=8, letters="XYZ+-", complex_coeffs=True)
    inp = sv.init_basis_state(n, 5)
    rep = sv.non_hermitian_gradient(circ, theta, obs, inp)
    vals, energy, _ = oracle.non_hermitian_values(circ, theta, obs, inp.amplitudes)
    assert max_err(rep.values, vals) <= GRAD_TOL
    assert abs(rep.energy - energy) <= ENERGY_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n", [(4, 22), (3, 20), (5, 21)])
def test_chunked_host_input_pipelines_leading_forward_passes(cfg, n, monkeypatch):
    """Large host inputs are copied in 16 chunks with the leading forward passes (tile
    qubits below the chunk boundary) launched chunk by chunk behind the copy: same
    kernels, same tiles -- the result is bitwise the one of the plain copy, and matches
    the oracle.  (The threshold, 26 qubits, is lowered through the test hook.)"""
    from cases import random_amplitudes
    from oracle import oracle

    w = sv.build_workload(cfg, n)
    inp = sv.StateVector(n, random_amplitudes(n, 17))
    monkeypatch.delenv("SVGB_CHUNK_MIN_QUBITS", raising=False)
    plain = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp)
    monkeypatch.setenv("SVGB_CHUNK_MIN_QUBITS", "16")
    chunked = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp)
    again = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp)
    assert np.array_equal(chunked.values, plain.values) and chunked.energy == plain.energy
    assert np.array_equal(again.values, plain.values)
    if n <= 20:
        vals, energy, _ = oracle.reverse_mode_values(w.circuit, w.theta, w.observable, inp.amplitudes)
        assert max_err(chunked.values, vals) <= GRAD_TOL
        assert abs(chunked.energy - energy) <= ENERGY_TOL
