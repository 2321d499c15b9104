"""GPU parity of the sharded engine (SURVEY.md §8 row e) on one device.

A virtual engine holds 2/4/8 shards of the state on one GPU and runs exactly
the distributed schedule of an NCCL job (top qubits = shard bits, rank-bit <->
local-qubit swaps, partner-shard fetches for observable terms that flip shard
bits, per-shard partial sums combined in shard order); only the exchange
transport differs (device copies instead of ncclSend/Recv).  Results must
meet the same bar as the single-shard engine against the reference's golden
outputs and the oracle.
"""
import numpy as np
import pytest

import paper_2009_02823_b200 as sv
from cases import config_cases, small_cases
from conftest import cvec, load_golden, materialize, max_err

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-10
ENERGY_TOL = 1e-12

GOLD = load_golden()
SMALL = {**small_cases(), **config_cases()}
_ENGINES: dict = {}


def _engine(shards):
    e = _ENGINES.get(shards)
    if e is None:
        e = _ENGINES[shards] = sv.distributed.virtual_engine(shards)
    return e


def _run(circ, theta, obs, inp, method, eng, stats=None):
    if method == "non_hermitian":
        return sv.non_hermitian_gradient(circ, theta, obs, inp, engine=eng)
    return sv.reverse_mode_gradient(circ, theta, obs, inp, engine=eng, stats=stats)


def _cases():
    out = []
    for name in sorted(SMALL):
        circ, _, _, _, _ = materialize(SMALL[name])
        for shards in (2, 4, 8):
            if circ.num_qubits - (shards.bit_length() - 1) >= 2:  # 2-qubit gates need 2 local qubits
                out.append((name, shards))
    return out


@pytest.mark.parametrize("name,shards", _cases())
def test_virtual_shards_match_reference_golden(name, shards):
    rec = GOLD[name]
    circ, theta, obs, inp, method = materialize(SMALL[name])
    rep = _run(circ, theta, obs, inp, method, _engine(shards))
    assert max_err(rep.values, cvec(rec["values"])) <= GRAD_TOL
    assert abs(rep.energy - complex(*rec["energy"])) <= ENERGY_TOL
    assert vars(rep.counters) == rec["counters"]


@pytest.mark.parametrize("shards", [2, 4, 8])
@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("name", ["cfg5_n15", "cfg4_n16", "cfg3_n14", "cfg2_n12"])
def test_virtual_shards_both_kernel_families(name, kernel, shards):
    """Tiles narrower than the shard (register and shared-memory kernels) with swaps."""
    rec = GOLD[name]
    circ, theta, obs, inp, _ = materialize(SMALL[name])
    eng = _engine(shards)
    eng.set_option("kernel", kernel)
    stats = {}
    try:
        rep = sv.reverse_mode_gradient(circ, theta, obs, inp, engine=eng, stats=stats)
    finally:
        eng.set_option("kernel", 0)
    assert max_err(rep.values, cvec(rec["values"])) <= GRAD_TOL
    assert abs(rep.energy - complex(*rec["energy"])) <= ENERGY_TOL
    assert stats["swaps"] > 0 and stats["exchange_bytes"] > 0


@pytest.mark.parametrize("shards", [2, 4])
@pytest.mark.parametrize("method", ["reverse", "non_hermitian"])
def test_virtual_shards_every_gate_kind(shards, method):
    """Dense and controlled gates, complex generators and global-flip observable terms."""
    from cases import all_kinds_circuit, mixed_observable, random_amplitudes
    from oracle import oracle

    n = 12
    circ = all_kinds_circuit(sv, n)
    theta = np.random.default_rng([7, n]).uniform(-np.pi, 2 * np.pi, circ.num_params)
    complex_obs = method == "non_hermitian"
    obs = mixed_observable(sv, n, 33, count=12, letters="XYZ+-" if complex_obs else "XYZH", complex_coeffs=complex_obs)
    inp = sv.StateVector(n, random_amplitudes(n, 4))
    eng = _engine(shards)
    for tile in (0, 8, 9):
        eng.set_option("tile_qubits", tile)
        try:
            rep = _run(circ, theta, obs, inp, method, eng)
        finally:
            eng.set_option("tile_qubits", 0)
        if complex_obs:
            vals, energy, _ = oracle.non_hermitian_values(circ, theta, obs, inp.amplitudes)
        else:
            vals, energy, _ = oracle.reverse_mode_values(circ, theta, obs, inp.amplitudes)
        assert max_err(rep.values, vals) <= GRAD_TOL, tile
        assert abs(rep.energy - energy) <= ENERGY_TOL


@pytest.mark.parametrize("shards", [2, 8])
def test_virtual_shards_wide_flip_terms(shards):
    """hadamard_all: Pauli strings flipping every qubit, shard bits included (partner fetch)."""
    from oracle import oracle

    n = 13
    circ = sv.Circuit(n, tuple(sv.ry(q, q) for q in range(n)) + tuple(sv.cx(q, (q + 1) % n) for q in range(n)), n)
    theta = np.linspace(0.1, 2.9, n)
    obs = sv.builtin_observable("hadamard_all", n)
    inp = sv.init_basis_state(n)
    rep = sv.reverse_mode_gradient(circ, theta, obs, inp, engine=_engine(shards))
    vals, energy, _ = oracle.reverse_mode_values(circ, theta, obs, inp.amplitudes)
    assert max_err(rep.values, vals) <= GRAD_TOL
    assert abs(rep.energy - energy) <= ENERGY_TOL


@pytest.mark.parametrize("cfg,n", [(3, 22), (4, 22), (5, 21)])
@pytest.mark.parametrize("shards", [2, 8])
def test_virtual_shards_match_single_shard_midsize(cfg, n, shards):
    w = sv.build_workload(cfg, n)
    inp = sv.BasisState(n)
    ref = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp)
    rep = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp, engine=_engine(shards))
    assert max_err(rep.values, ref.values) <= GRAD_TOL
    assert abs(rep.energy - ref.energy) <= ENERGY_TOL


@pytest.mark.parametrize("cfg", [3, 5])
def test_sharded_wide_tiles_match_single_shard(cfg):
    """Shards of >= 24 qubits: 12-qubit tiles, free-lane layouts and carried scales in
    the generated kernels, with swaps through the NCCL data path (emulated)."""
    n = 25
    w = sv.build_workload(cfg, n)
    inp = sv.BasisState(n)
    ref = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp)
    eng = sv.distributed.virtual_engine(2)
    eng.set_option("emulate_transport", 1)
    stats = {}
    rep = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp, engine=eng, stats=stats)
    assert stats["tile_qubits"] == 12 and stats["jit_passes"] > 0
    assert max_err(rep.values, ref.values) <= GRAD_TOL
    assert abs(rep.energy - ref.energy) <= ENERGY_TOL


def test_virtual_shards_expectation_and_determinism():
    circ, theta, obs, inp, _ = materialize(SMALL["cfg5_n15"])
    eng = _engine(4)
    e = sv.circuit_expectation(circ, theta, obs, inp, engine=eng)
    assert abs(e - complex(*GOLD["cfg5_n15"]["energy"])) <= ENERGY_TOL
    a = sv.reverse_mode_gradient(circ, theta, obs, inp, engine=eng)
    b = sv.reverse_mode_gradient(circ, theta, obs, inp, engine=eng)
    assert np.array_equal(a.values, b.values) and a.energy == b.energy


@pytest.mark.parametrize("shards", [2, 4, 8])
@pytest.mark.parametrize("name", ["cfg5_n15", "cfg4_n16", "cfg3_n14", "nh_all_kinds_6", "cfg2_n12"])
def test_nccl_data_path_emulated(name, shards):
    """The NCCL engine's own data path -- half-shard pack, exchange, unpack for qubit
    swaps; partner shard fetched into the scratch buffer for shard-flipping terms --
    with device copies standing in for ncclSend/ncclRecv."""
    rec = GOLD[name]
    circ, theta, obs, inp, method = materialize(SMALL[name])
    if circ.num_qubits - (shards.bit_length() - 1) < 2:
        pytest.skip("shard too small")
    eng = sv.distributed.virtual_engine(shards)
    eng.set_option("emulate_transport", 1)
    rep = _run(circ, theta, obs, inp, method, eng)
    assert max_err(rep.values, cvec(rec["values"])) <= GRAD_TOL
    assert abs(rep.energy - complex(*rec["energy"])) <= ENERGY_TOL


@pytest.mark.parametrize("name", ["cfg5_n15", "cfg3_n14", "nh_all_kinds_6"])
def test_nccl_engine_single_rank(name):
    """The NCCL engine on one GPU (one-rank communicator): NCCL loading, communicator
    setup and the result all-gather run for real; exchanges need >= 2 ranks."""
    from paper_2009_02823_b200 import _native

    rec = GOLD[name]
    circ, theta, obs, inp, method = materialize(SMALL[name])
    eng = _native.Engine(0, shards=1, rank=0, nccl_id=_native.nccl_unique_id())
    rep = _run(circ, theta, obs, inp, method, eng)
    assert max_err(rep.values, cvec(rec["values"])) <= GRAD_TOL
    assert abs(rep.energy - complex(*rec["energy"])) <= ENERGY_TOL


@pytest.mark.parametrize("name", ["cfg5_n15", "cfg3_n14"])
def test_nccl_engine_single_rank_slice_input(name):
    """A dense host input handed to an NCCL rank as its ShardSlice (SVG_FLAG_INPUT_LOCAL):
    one rank of one -> the slice is the whole state; same result as the StateVector."""
    from paper_2009_02823_b200 import _native

    rec = GOLD[name]
    circ, theta, obs, inp, method = materialize(SMALL[name])
    eng = _native.Engine(0, shards=1, rank=0, nccl_id=_native.nccl_unique_id())
    dense = sv.StateVector(circ.num_qubits, inp.amplitudes)
    sl = sv.ShardSlice(circ.num_qubits, np.array(inp.amplitudes), 0, 1)
    a = sv.reverse_mode_gradient(circ, theta, obs, dense, engine=eng)
    b = sv.reverse_mode_gradient(circ, theta, obs, sl, engine=eng)
    assert np.array_equal(a.values, b.values) and a.energy == b.energy
    assert max_err(b.values, cvec(rec["values"])) <= GRAD_TOL
    with pytest.raises(ValueError, match="slice"):
        sv.reverse_mode_gradient(circ, theta, obs, sv.ShardSlice(circ.num_qubits, np.array(
            inp.amplitudes[: len(inp.amplitudes) // 2]), 1, 2), engine=eng)


@pytest.mark.slow
def test_cfg5_structure_n30_eight_virtual_shards_vs_oracle_fixture():
    """cfg 5's structure (RX/RY/RZ + RZZ chain, 128 random Pauli strings) at n = 30 over
    8 virtual shards with the NCCL data path emulated (half-shard pack/exchange/unpack,
    partner fetches), against the full-size oracle fixture (tests/golden/make_oracle_n30.py):
    every entry <= 1e-10 abs-or-rel, energy <= 1e-12."""
    gold = load_golden("oracle_cfg5_n30.json")["cfg5_n30"]
    w = sv.build_workload(5, 30)
    eng = sv.distributed.virtual_engine(8)
    eng.set_option("emulate_transport", 1)
    stats = {}
    rep = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, sv.BasisState(30), engine=eng, stats=stats)
    eng.close()
    assert stats["swaps"] >= 1
    assert max_err(rep.values, np.asarray(gold["values_real"], dtype=complex)) <= GRAD_TOL
    assert abs(rep.energy - complex(*gold["energy"])) <= ENERGY_TOL
    assert vars(rep.counters) == gold["counters"]
