"""Checked generated kernels (in place of compute-sanitizer, which this GPU pool does not
run): with the engine option ``checked`` every shared-memory element a generated
kernel reads is overwritten with a NaN right after the read, and every global tile
index is bounds-checked (``__trap``).  A read that comes before its write in a later
phase -- a missing barrier or cp.async wait, a wrong swizzle, a staging slot reused
too early -- then returns NaN and fails the parity check (or the numeric guard); an
out-of-range tile address traps.  Covered: free-lane layouts with swizzled
transposes and tile-order staging, private-slice staging, shared-memory segments,
R = 3 / 4, tiles of 7..12 qubits, several tiles per CTA, the PDL chain."""
import numpy as np
import pytest

import paper_2009_02823_b200 as sv
from cases import config_cases, small_cases
from conftest import cvec, load_golden, materialize, max_err

pytestmark = pytest.mark.gpu
GOLD = load_golden()
CASES = {**small_cases(), **config_cases()}


@pytest.mark.parametrize("name,tile,reg_bits", [("cfg3_n14", 9, 4), ("cfg3_n14", 10, 3), ("cfg5_n15", 10, 4),
                                                ("cfg4_n16", 12, 4), ("cfg2_n12", 8, 3), ("cfg1", 0, 0),
                                                ("family_D9_random", 9, 4), ("cfg5_n15", 8, 3)])
def test_checked_generated_kernels(name, tile, reg_bits):
    rec = GOLD[name]
    circ, theta, obs, inp, _ = materialize(CASES[name])
    eng = sv._native.engine()
    opts = {"jit": 2, "checked": 1, "tile_qubits": tile, "reg_bits": reg_bits}
    try:
        for k, v in opts.items():
            eng.set_option(k, v)
        stats = {}
        rep = sv.reverse_mode_gradient(circ, theta, obs, inp, stats=stats)
    finally:
        for k, v in {"jit": 1, "checked": 0, "tile_qubits": 0, "reg_bits": 0}.items():
            eng.set_option(k, v)
    assert stats["jit_passes"] > 0 and stats["nonfinite"] == 0
    assert np.all(np.isfinite(rep.values))
    assert max_err(rep.values, cvec(rec["values"])) <= 1e-10
    assert abs(rep.energy - complex(*rec["energy"])) <= 1e-12


def test_checked_full_size_cfg3_pass():
    """cfg 3 at n = 26 (12-qubit tiles, 1 CTA per SM, many tiles per CTA) in checked mode."""
    rec = load_golden("golden_cfg3.json")["cfg3"]
    from cases import large_config_cases

    circ, theta, obs, inp, _ = materialize(large_config_cases()["cfg3"])
    eng = sv._native.engine()
    eng.set_option("checked", 1)
    try:
        rep = sv.reverse_mode_gradient(circ, theta, obs, inp)
    finally:
        eng.set_option("checked", 0)
    assert max_err(rep.values, cvec(rec["values"])) <= 1e-10
