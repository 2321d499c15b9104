"""One small gradient through the generated kernels, for compute-sanitizer (tests/test_gpu_sanitizer.py).

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tests/sanitize_case.py NAME TILE

Runs golden case NAME with circuit-specialised kernels forced on (jit=2) and the
given tile width (free-lane layouts, swizzled transposes, cp.async staging into
reused buffers, the PDL chain between passes), checks it against the golden
values and exits 0; any sanitizer report makes compute-sanitizer exit non-zero.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

import paper_2009_02823_b200 as sv  # noqa: E402
from cases import config_cases, small_cases  # noqa: E402
from conftest import cvec, load_golden, materialize, max_err  # noqa: E402


def main():
    name, tile = sys.argv[1], int(sys.argv[2])
    rec = load_golden()[name]
    circ, theta, obs, inp, _ = materialize({**small_cases(), **config_cases()}[name])
    eng = sv._native.engine()
    eng.set_option("jit", 2)
    eng.set_option("tile_qubits", tile)
    stats = {}
    rep = sv.reverse_mode_gradient(circ, theta, obs, inp, stats=stats)
    err = max_err(rep.values, cvec(rec["values"]))
    assert err <= 1e-10, err
    assert abs(rep.energy - complex(*rec["energy"])) <= 1e-12
    assert stats["jit_passes"] > 0
    print(f"ok {name} tile={tile} err={err:.1e} jit_passes={stats['jit_passes']} segments={stats['segments']}")


if __name__ == "__main__":
    main()
