"""CPU-only checks of the host side: C-ABI surface, table layouts, lowering, planner."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2009_02823_b200 as sv
from cases import config_cases, small_cases
from conftest import ROOT, cvec, gpu_available, load_golden, materialize, max_err
from emulator import emulate
from paper_2009_02823_b200 import _native, lowering

GOLD = load_golden()
CASES = {**small_cases(), **config_cases()}


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "svgrad_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(svg_\w+)\(", header, flags=re.M))
    assert declared == set(_native.EXPORTED)
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert _native.load().svg_abi_version() == _native.ABI_VERSION


@pytest.mark.parametrize("dtype,ctype", [
    (lowering.GATE_DTYPE, _native.svg_gate),
    (lowering.DERIV_DTYPE, _native.svg_deriv),
    (lowering.TERM_DTYPE, _native.svg_pauli_term),
])
def test_numpy_tables_match_c_layout(dtype, ctype):
    assert dtype.itemsize == ctypes.sizeof(ctype)
    for name, _ in ctype._fields_:
        assert dtype.fields[name][1] == getattr(ctype, name).offset, name


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_no_silent_cpu_fallback():
    circ = sv.Circuit(1, (sv.ry(0, 0),), 1)
    with pytest.raises(sv.NativeUnavailable):
        sv.reverse_mode_gradient(circ, [0.3], sv.Observable(1, ((1.0, "Z"),)), sv.init_basis_state(1))


EMULATED = [n for n in sorted(CASES) if GOLD[n]["num_qubits"] <= 12 and GOLD[n]["method"] == "reverse"]


@pytest.mark.parametrize("name", EMULATED)
def test_lowered_tables_reproduce_reference(name):
    """Binding + generators + planner order + accumulation order, executed densely."""
    rec = GOLD[name]
    circ, theta, obs, inp, _ = materialize(CASES[name])
    sums, energy, _ = emulate(circ, theta, obs, inp, tile_qubits=0)
    assert max_err(2 * sums.real, cvec(rec["values"]).real) <= 1e-10
    assert abs(energy - complex(*rec["energy"])) <= 1e-12


@pytest.mark.parametrize("name,tile", [("cfg3_n14", 7), ("cfg5_n11", 7), ("cfg4_n12", 8), ("all_kinds_6_random", 7)])
def test_planner_reordering_is_exact(name, tile):
    rec = GOLD[name]
    circ, theta, obs, inp, _ = materialize(CASES[name])
    sums, energy, (order, start, qmasks, k) = emulate(circ, theta, obs, inp, tile_qubits=tile)
    assert max_err(2 * sums.real, cvec(rec["values"]).real) <= 1e-10
    assert sorted(order.tolist()) == list(range(len(circ.gates)))
    prob = lowering.Problem(circ, theta, obs, inp)
    for p in range(len(qmasks)):
        q = int(qmasks[p])
        assert bin(q).count("1") == min(k, circ.num_qubits)
        for gi in order[start[p]: start[p + 1]]:
            g = prob.gates[gi]
            flip = int(g["x_mask"]) if g["form"] == _native.FORM_PAULI else sum(1 << t for t in g["targets"][: g["ntargets"]])
            assert flip & ~q == 0


def test_plan_fuses_full_size_configs():
    """Pass counts at BASELINE sizes (host planning only, no allocation)."""
    for cfg in (2, 3, 4, 5):
        w = sv.build_workload(cfg)
        prob = lowering.Problem(w.circuit, w.theta, w.observable, sv.BasisState(w.num_qubits))
        order, start, qmasks, k = _native.plan_inspect(prob.c, 0, 148)
        passes = len(start) - 1
        assert passes < w.num_gates / 4, (cfg, passes)


def test_window_planner_cuts_hbm_passes():
    """The engine's plan at full size without a GPU (svg_debug_plan_stats): passes over
    windows of contiguous qubits hold parallelograms of the layered circuits, so
    cfg 4 (n = 30) needs about half the HBM passes of the layer-by-layer greedy plan,
    no pass exceeds the per-thread accumulator budget, and every gate is placed once."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from plan_stats import stats

    new, old = stats(4, None, windows=1), stats(4, None, windows=0)
    for d in ("fwd", "rev"):
        assert new[d]["reg_ops"] == old[d]["reg_ops"] == new["gates"] == 1424
        assert new[d]["passes"] <= 30 < 50 <= old[d]["passes"], (new[d], old[d])
    assert new["rev"]["lane_group_acc"] == 0 and new["rev"]["max_slots"] <= 46
    c3 = stats(3, None, windows=1)
    assert c3["rev"]["passes"] <= 48 and c3["rev"]["lane_group_acc"] == 0


@pytest.mark.parametrize("k,regbits,lowb", [(12, 4, 4), (11, 4, 5), (12, 3, 4), (10, 4, 3)])
def test_free_lane_segment_plans_are_valid(k, regbits, lowb):
    """Beam-search segment planner (plan_segments_free) on random passes of one-qubit-flip
    gates: every gate lands in exactly one segment, flips only register positions of its
    segment, conflicting gates keep their order, and the layouts are well formed."""
    import ctypes as C

    from paper_2009_02823_b200 import _native as N

    lib = N.load()
    rng = np.random.default_rng([k, regbits, lowb])
    for trial in range(12):
        m = int(rng.integers(1, 70))
        width = int(rng.integers(2, k + 1))  # active tile positions of this pass
        active = rng.choice(k, size=width, replace=False)
        flips = np.zeros(m, dtype=np.uint32)
        touch = np.zeros(m, dtype=np.uint32)
        for i in range(m):
            kind = rng.integers(0, 3)
            t = int(rng.choice(active))
            if kind == 0:      # rotation with a flip
                flips[i] = touch[i] = 1 << t
            elif kind == 1:    # diagonal
                touch[i] = 1 << t
            else:              # controlled flip: control is diagonal
                c = int(rng.choice(active))
                flips[i] = 1 << t
                touch[i] = (1 << t) | (1 << c)
        seg = np.zeros(m, dtype=np.int32)
        pos = np.zeros(m, dtype=np.int32)
        regmask = np.zeros(m + 1, dtype=np.uint32)
        lanemask = np.zeros(m + 1, dtype=np.uint32)
        nsegs = C.c_int32()
        rc = lib.svg_debug_segments(flips.ctypes.data_as(C.c_void_p), touch.ctypes.data_as(C.c_void_p), m, k, regbits, lowb,
                                    seg.ctypes.data_as(C.c_void_p), pos.ctypes.data_as(C.c_void_p),
                                    regmask.ctypes.data_as(C.c_void_p), lanemask.ctypes.data_as(C.c_void_p),
                                    C.byref(nsegs))
        assert rc == 0, lib.svg_last_error()
        ns = nsegs.value
        assert 1 <= ns <= m and (seg >= 0).all() and (seg < ns).all()
        assert len({(int(a), int(b)) for a, b in zip(seg, pos)}) == m
        for s_ in range(ns):
            r, l = int(regmask[s_]), int(lanemask[s_])
            assert bin(r).count("1") == regbits and bin(l).count("1") == 5 and r & l == 0 and (r | l) < (1 << k)
        for i in range(m):
            assert int(flips[i]) & ~int(regmask[seg[i]]) == 0
            for j in range(i + 1, m):
                if int(touch[i]) & int(touch[j]) & (int(flips[i]) | int(flips[j])):
                    assert (seg[i], pos[i]) < (seg[j], pos[j]), (trial, i, j)


def test_pauli_lowering_of_rotations():
    """a I + b P of the tables equals the reference closed form cos(at) I + i sin(at) P."""
    from paper_2009_02823_b200.ir import bound_matrix, pauli_product

    theta = np.array([0.37, -1.2])
    circ = sv.Circuit(3, (sv.rp("XY", (0, 2), 0), sv.cry(1, 2, 1, alpha=0.8)), 2)
    gates, derivs = lowering.bind(circ, theta)
    for i, g in enumerate(circ.gates):
        P = pauli_product(g.kind.axes)
        U = gates[i]["fwd"][0] * np.eye(P.shape[0]) + gates[i]["fwd"][1] * P
        assert np.allclose(U, bound_matrix(g, theta), atol=1e-15)
        R = gates[i]["rewind"][0] * np.eye(P.shape[0]) + gates[i]["rewind"][1] * P
        assert np.allclose(R @ U, np.eye(P.shape[0]), atol=1e-15)
        K = derivs[i]["k"][0] * np.eye(P.shape[0]) + derivs[i]["k"][1] * P
        # reference derivative action: sigma per axis, then the bound rotation, scalar alpha*i,
        # acting on phi_i; the table holds it in the post-gate basis: K' = K_pre U^-1
        assert derivs[i]["basis"] == 1
        assert np.allclose(K @ U, g.kind.alpha * 1j * (U @ P), atol=1e-15)


def test_non_pauli_observable_letters_expand_exactly():
    from paper_2009_02823_b200.operators import dense_matrix, pauli_strings
    from paper_2009_02823_b200.ir import pauli_product

    obs = sv.Observable(3, ((0.7, "H+-"), (1.5j, "-ZH"), (-0.2, "IIY")))
    dense = np.zeros((8, 8), dtype=complex)
    for s in pauli_strings(obs):
        letters = "".join("Y" if (s.x_mask >> q) & (s.z_mask >> q) & 1 else "X" if (s.x_mask >> q) & 1
                          else "Z" if (s.z_mask >> q) & 1 else "I" for q in range(3))
        dense += s.coeff * pauli_product(letters)
    assert np.allclose(dense, dense_matrix(obs), atol=1e-15)


@pytest.mark.parametrize("cfg,n,tile,checked", [(2, 14, 0, 0), (3, 20, 12, 0), (5, 18, 0, 0), (3, 16, 10, 1)])
def test_generated_kernels_compile_for_sm100a(cfg, n, tile, checked):
    """Without a GPU: lower the config with circuit-specialised kernels forced on and
    NVRTC-compile every distinct generated pass kernel for sm_100a (free-lane
    layouts, swizzled transposes, tile-order staging, fused diagonal runs)."""
    import ctypes as C

    from paper_2009_02823_b200 import _native as N
    from paper_2009_02823_b200.lowering import Problem

    lib = N.load()
    w = sv.build_workload(cfg, n)
    pr = Problem(w.circuit, w.theta, w.observable, sv.BasisState(n), real_sums=True)
    opts = (C.c_int64 * 4)(tile, 0, checked, 0)
    count = C.c_int32()
    rc = lib.svg_debug_jit_check(C.byref(pr.c), opts, C.byref(count))
    if rc != 0 and (b"NVRTC" in (lib.svg_last_error() or b"") or b"libnvrtc" in (lib.svg_last_error() or b"")):
        pytest.skip("libnvrtc not present")
    assert rc == 0, lib.svg_last_error()
    assert count.value > 0


def test_numeric_guard_rules():
    """NaN/Inf device sums: raise only when the inputs cannot explain them (finite
    tables and input, unitary gates); otherwise pass them through as numpy would."""
    from paper_2009_02823_b200.adjoint import _numeric_guard
    from paper_2009_02823_b200.lowering import Problem

    w = sv.build_workload(1, 6)
    pr = Problem(w.circuit, w.theta, w.observable, sv.BasisState(6))
    with pytest.raises(FloatingPointError, match="device fault"):
        _numeric_guard(w.circuit, pr, 3)
    theta = w.theta.copy()
    theta[2] = np.nan
    pr_nan = Problem(w.circuit, theta, w.observable, sv.BasisState(6))
    _numeric_guard(w.circuit, pr_nan, 3)  # NaN input: the reference propagates it too
    nu = sv.Gate(sv.NonUnitary(lambda: np.diag([1e300, 1.0]), 0), (0,))
    circ = sv.Circuit(6, (*w.circuit.gates, nu), w.circuit.num_params)
    _numeric_guard(circ, Problem(circ, w.theta, w.observable, sv.BasisState(6)), 1)  # may overflow: allowed
