"""Parity cases shared by the golden-fixture generator and the tests.

Every builder takes an ``api`` namespace exposing the reference's public
names (``svgrad`` in this container when generating fixtures; this package's
``paper_2009_02823_b200`` in the tests), so fixture and test build the same
circuit from the same code.  The cases follow the reference's own pins:

* analytic single-Ry (``pkg/tests/test_gradients.py:45-51``),
* the oracle triangle over ansatz families A-D x N=3..5 with hadamard_all
  (``pkg/tests/test_gradients.py:131-144``; families ``svgrad/ansatz.py:1-88``),
* repeated / multi-parameter / shared-slot gates (``:85-126``, ``:174-195``),
* NonUnitary gates (``:204-214``), random input states (``:362-377``),
* every gate kind and derivative rule (``pkg/tests/test_circuit.py:210-233``),
* non-Hermitian operators (``pkg/tests/test_gradients.py:226-267``),
* BASELINE.json cfg 1-5 at full and reduced size (``configs.py``).
"""
from __future__ import annotations

import numpy as np

TWO_PI = 2.0 * np.pi


# -- matrices used by callable gate kinds (own closed forms, numpy only) -------

def _rz(t):
    return np.diag([np.exp(-0.5j * t), np.exp(0.5j * t)])


def _ry(t):
    c, s = np.cos(t / 2), np.sin(t / 2)
    return np.array([[c, -s], [s, c]], dtype=complex)


def two_angle_matrix(a, b):
    return _rz(b) @ _ry(a)


def two_angle_derivative(which, a, b):
    if which == 0:
        c, s = np.cos(a / 2), np.sin(a / 2)
        return _rz(b) @ (0.5 * np.array([[-s, -c], [c, -s]], dtype=complex))
    return (np.diag([-0.5j, 0.5j]) @ _rz(b)) @ _ry(a)


def scaled_ry(t):
    return np.diag([1.0, 2.0]) @ _ry(t)


def xy_coupler(t):
    """4x4 iSWAP-like exchange, sub-index bit k <-> targets[k]."""
    c, s = np.cos(t), np.sin(t)
    return np.array(
        [[1, 0, 0, 0], [0, c, -1j * s, 0], [0, -1j * s, c, 0], [0, 0, 0, np.exp(0.3j * t)]],
        dtype=complex,
    )


def scaled_coupler(t):
    return np.diag([1.0, 0.5, 1.5, 1.0]) @ xy_coupler(t)


# -- ansatz families A-D (restated from the docstring of svgrad/ansatz.py) ------

def family_circuit(api, family: str, n: int, reps: int):
    gates, p = [], 0

    def take():
        nonlocal p
        p += 1
        return p - 1

    if family in "AB":
        for _ in range(reps):
            gates += [api.rx(q, take()) for q in range(n)]
            gates += [api.rz(q, take()) for q in range(n)]
            if family == "B":
                gates += [api.cx(k + 1, k) for k in range(n - 2, -1, -1)]
    elif family == "C":
        gates += [api.ry(q, take()) for q in range(n)]
        gates += [api.rz(q, take()) for q in range(n)]
        for _ in range(reps):
            gates += [api.cx(k, k + 1) for k in range(n - 1)]
            gates += [api.ry(q, take()) for q in range(n)]
            gates += [api.rz(q, take()) for q in range(n)]
    else:
        for layer in range(reps):
            gates += [api.ry(q, take()) for q in range(n)]
            for j in range(n):
                a, b = (j + layer) % n, (j + layer + 1) % n
                c, t = (a, b) if layer % 2 == 0 else (b, a)
                gates.append(api.crx(c, t, take()))
    return api.Circuit(n, tuple(gates), p)


def random_amplitudes(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng([seed, n, 77])
    amps = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return amps / np.linalg.norm(amps)


def input_state(api, n: int, spec):
    """spec: ("basis", index) or ("random", seed)."""
    kind, value = spec
    if kind == "basis":
        return api.init_basis_state(n, value)
    return api.StateVector(n, random_amplitudes(n, value))


def _z(n, placed):
    return "".join(placed.get(q, "I") for q in range(n))


def mixed_observable(api, n: int, seed: int, count: int = 8, letters: str = "XYZ", complex_coeffs=False):
    rng = np.random.default_rng([seed, n, 5])
    terms = []
    for _ in range(count):
        w = int(rng.integers(1, min(n, 4) + 1))
        qs = rng.choice(n, size=w, replace=False)
        ls = rng.integers(0, len(letters), size=w)
        c = float(rng.normal())
        if complex_coeffs:
            c = complex(c, float(rng.normal()))
        terms.append((c, _z(n, {int(q): letters[int(l)] for q, l in zip(qs, ls)})))
    return api.Observable(n, tuple(terms))


def all_kinds_circuit(api, n: int, controlled_matrix: bool = True):
    """Every gate kind and derivative rule, controls included, repeated params."""
    G, K = api.Gate, api
    gates = [
        api.fixed("h", 0), api.fixed("h", n - 1), api.rx(0, 0), api.ry(1, 1), api.rz(2 % n, 2),
        api.cx(0, 1), api.crx(1, 2 % n, 3), api.cry(2 % n, 0, 4), api.crz(0, n - 1, 5),
        api.rp("XY", (0, 2 % n), 6), api.rp("ZZ", (1, n - 1), 7), api.rp("YX", (n - 1, 1), 8),
        api.phase_gate(1, 9), api.fixed("y", 2 % n), api.fixed("z", 0),
        G(K.PauliRotation("X", alpha=0.75), (n - 1,), (0,), (10,)),
        G(K.CustomParametric(two_angle_matrix, 2, derivative_fn=two_angle_derivative, name="zy"), (1,), (), (11, 12)),
        G(K.CustomParametric(two_angle_matrix, 2, name="zy-fd"), (2 % n,), (0,) if controlled_matrix else (), (13, 13)),
        G(K.CustomParametric(xy_coupler, 1, name="xy"), (2 % n, 0), (), (14,)),
        G(K.NonUnitary(scaled_ry, 1, name="scaled-ry"), (0,), (), (15,)),
        G(K.NonUnitary(scaled_coupler, 1, name="scaled-xy"), (1, n - 1), (), (16,)),
        api.ry(0, 17),
        api.rx(1, 0), api.rz(0, 2),  # repeated parameters
        G(K.Phase(), (0,), (1,), (18,)),
        G(K.PauliRotation("YY"), (0, 1), (2 % n,), (19,)) if n >= 3 else api.ry(0, 19),
    ]
    return api.Circuit(n, tuple(gates), 21)  # slot 20 unreferenced


# -- the case table ---------------------------------------------------------------
# Each case: (name, builder(api) -> dict(circuit, theta, obs, input, method)).

SINGLE_RY_THETAS = (0.0, 0.3, np.pi / 2, 2.0, np.pi, 5.1)


def _case(circuit, theta, obs, inp, method="reverse"):
    return dict(circuit=circuit, theta=np.asarray(theta, dtype=float), obs=obs, input=inp, method=method)


def small_cases():
    cases = {}
    for i, th in enumerate(SINGLE_RY_THETAS):
        cases[f"single_ry_{i}"] = lambda api, th=th: _case(
            api.Circuit(1, (api.ry(0, 0),), 1), [th], api.Observable(1, ((1.0, "Z"),)), ("basis", 0)
        )
    for fam in "ABCD":
        for n in (3, 4, 5):
            for draw in range(2):
                def build(api, fam=fam, n=n, draw=draw):
                    circ = family_circuit(api, fam, n, 2)
                    rng = np.random.default_rng([100 + n, draw, ord(fam)])
                    th = rng.uniform(0, TWO_PI, circ.num_params)
                    return _case(circ, th, api.builtin_observable("hadamard_all", n), ("basis", 0))
                cases[f"family_{fam}{n}_{draw}"] = build
    cases["repeated_rz"] = lambda api: _case(
        api.Circuit(1, (api.fixed("h", 0), api.rz(0, 0), api.rz(0, 0)), 1), [0.35],
        api.Observable(1, ((1.0, "X"),)), ("basis", 0))
    cases["unreferenced_slot"] = lambda api: _case(
        api.Circuit(1, (api.ry(0, 0),), 2), [0.4, 9.9], api.Observable(1, ((1.0, "Z"),)), ("basis", 0))
    cases["no_params"] = lambda api: _case(
        api.Circuit(2, (api.fixed("h", 0), api.cx(0, 1)), 0), [], api.builtin_observable("z_all", 2), ("basis", 0))
    cases["multi_param_fd"] = lambda api: _case(
        api.Circuit(2, (api.fixed("h", 0), api.Gate(api.CustomParametric(two_angle_matrix, 2, name="zy"), (0,), (), (0, 1)),
                        api.cx(0, 1), api.ry(1, 2)), 3),
        [0.7, -0.4, 1.9], api.builtin_observable("z_all", 2), ("basis", 0))
    cases["shared_slot"] = lambda api: _case(
        api.Circuit(1, (api.fixed("h", 0), api.Gate(api.CustomParametric(two_angle_matrix, 2, name="zy"), (0,), (), (0, 0))), 1),
        [0.6], api.Observable(1, ((1.0, "X"),)), ("basis", 0))
    cases["non_unitary"] = lambda api: _case(
        api.Circuit(2, (api.ry(0, 0), api.Gate(api.NonUnitary(scaled_ry, 1, name="scaled-ry"), (0,), (), (1,)),
                        api.cx(0, 1), api.rx(1, 2)), 3),
        [0.9, 0.3, -1.2], api.builtin_observable("z_all", 2), ("basis", 0))
    for n in (3, 4, 6):
        for inp in (("basis", 0), ("random", 3)):
            def build(api, n=n, inp=inp):
                circ = all_kinds_circuit(api, n)
                th = np.random.default_rng([7, n]).uniform(-np.pi, TWO_PI, circ.num_params)
                return _case(circ, th, mixed_observable(api, n, 11, letters="XYZH"), inp)
            cases[f"all_kinds_{n}_{inp[0]}"] = build
    cases["random_input_family_C"] = lambda api: _case(
        family_circuit(api, "C", 3, 1), np.random.default_rng(45).uniform(0, TWO_PI, 12),
        api.builtin_observable("hadamard_all", 3), ("random", 45))
    for n in (7, 9):
        def build(api, n=n):
            circ = family_circuit(api, "D", n, 3)
            th = np.random.default_rng([n, 9]).uniform(0, TWO_PI, circ.num_params)
            return _case(circ, th, mixed_observable(api, n, 12, count=20), ("random", n))
        cases[f"family_D{n}_random"] = build
    # non-Hermitian operators (pkg/tests/test_gradients.py:226-267)
    for i, th in enumerate((0.0, 0.4, 1.3, 2.9)):
        cases[f"nh_lowering_{i}"] = lambda api, th=th: _case(
            api.Circuit(1, (api.ry(0, 0),), 1), [th], api.Observable(1, ((1.0, "-"),)), ("basis", 0), "non_hermitian")
    cases["nh_complex"] = lambda api: _case(
        api.Circuit(2, (api.ry(0, 0), api.phase_gate(0, 1), api.cx(0, 1), api.rx(1, 2)), 3),
        [0.8, 1.1, -0.6], api.Observable(2, ((1.0 + 0.5j, "-Z"), (0.25j, "XI"))), ("basis", 0), "non_hermitian")
    for n in (4, 6):
        def build(api, n=n):
            circ = all_kinds_circuit(api, n)
            th = np.random.default_rng([8, n]).uniform(-np.pi, TWO_PI, circ.num_params)
            return _case(circ, th, mixed_observable(api, n, 13, letters="XYZH+-", complex_coeffs=True),
                         ("random", n), "non_hermitian")
        cases[f"nh_all_kinds_{n}"] = build
    return cases


def config_cases():
    """BASELINE.json configs: full size where the reference finishes in seconds, else reduced n."""
    from paper_2009_02823_b200.configs import build_workload

    out = {}
    for cfg, n in ((1, None), (2, 12), (3, 10), (3, 14), (4, 12), (4, 16), (5, 11), (5, 15)):
        name = f"cfg{cfg}" + ("" if n is None else f"_n{n}")

        def build(api, cfg=cfg, n=n):
            w = build_workload(cfg, n, api=api)
            return _case(w.circuit, w.theta, w.observable, ("basis", 0))
        out[name] = build
    return out


def large_config_cases():
    """Reference runs that take seconds to an hour (generated separately)."""
    from paper_2009_02823_b200.configs import build_workload

    out = {}
    for cfg, n in ((2, None), (3, 20), (4, 20), (5, 20), (3, None)):
        name = f"cfg{cfg}" + ("" if n is None else f"_n{n}")

        def build(api, cfg=cfg, n=n):
            w = build_workload(cfg, n, api=api)
            return _case(w.circuit, w.theta, w.observable, ("basis", 0))
        out[name] = build
    return out
