"""Full-size (n = 30) oracle fixtures for the configs the reference cannot run.

    python tests/golden/make_oracle_n30.py cfg4        # BASELINE cfg 4 at its full size (n = 30)
    python tests/golden/make_oracle_n30.py cfg5_n30    # cfg 5's structure (12 layers RX/RY/RZ + RZZ chain,
                                                       # 128 random Pauli strings) at n = 30
    python tests/golden/make_oracle_n30.py hadamard_n26  # cfg 4's structure at n = 26 under hadamard_all

The reference needs ~0.5 TiB and ~5 h for cfg 4 and cannot hold cfg 5 at all
(SURVEY.md §8(c)), so these fixtures come from the C oracle
(oracle/svgrad_oracle.c, ``oracle_sweep_lean``: the literal schedule of
svgrad/gradients.py:128-173 with the derivative probe contracted group by
group instead of materialised).  The oracle itself is pinned to the
reference's own outputs on every golden case, including cfg 3 at its full
size (tests/test_oracle.py), and the lean variant is pinned to the literal
one (tests/test_oracle.py::test_lean_sweep_matches_literal).

Runs on the CPU only (any host with >= 48 GiB free; it is test infrastructure,
never the product path).  Output: tests/golden/oracle_<name>.json with the
gradient values (2 Re of the sums, as reverse_mode_gradient reports them),
the energy, the OpCounters, a structural digest of the workload, the oracle
source's sha256 and the wall time.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from golden.digest import circuit_digest, obs_digest  # noqa: E402

# name -> (config, qubits, observable override): hadamard_n26 is cfg 4's circuit structure at
# n = 26 under the paper's benchmark operator hadamard_all (one product term of 26 H factors)
CASES = {"cfg4": (4, None, None), "cfg5_n30": (5, 30, None), "hadamard_n26": (4, 26, "hadamard_all")}


def workload(name):
    import paper_2009_02823_b200 as sv

    cfg, n, obs = CASES[name]
    w = sv.build_workload(cfg, n)
    if obs:
        w = type(w)(w.cfg, w.num_qubits, w.circuit, sv.builtin_observable(obs, w.num_qubits), w.theta)
    return w


def main():
    name = sys.argv[1]
    threads = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    from oracle import oracle

    w = workload(name)
    with open(oracle.SRC, "rb") as f:
        src_sha = hashlib.sha256(f.read()).hexdigest()
    t0 = time.perf_counter()
    r = oracle.sweep_lean(w.circuit, w.theta, w.observable, None, 0, threads=threads)
    dt = time.perf_counter() - t0
    values = 2.0 * r.sums.real
    rec = {
        "method": "reverse",
        "num_qubits": w.num_qubits,
        "num_gates": w.num_gates,
        "num_params": w.circuit.num_params,
        "num_terms": len(w.observable.terms),
        "circuit_digest": circuit_digest(w.circuit),
        "obs_digest": obs_digest(w.observable),
        "theta_sum": float(np.sum(w.theta)),
        "input": ["basis", 0],
        "values_real": [float(x) for x in values],
        "sums_imag_max": float(np.max(np.abs(r.sums.imag))) if len(r.sums) else 0.0,
        "energy": [r.energy.real, r.energy.imag],
        "counters": r.counters,
        "oracle": "oracle/svgrad_oracle.c oracle_sweep_lean",
        "oracle_sha256": src_sha,
        "threads": threads or oracle.max_threads(),
        "oracle_seconds": dt,
    }
    out = os.path.join(HERE, f"oracle_{name}.json")
    with open(out, "w") as f:
        json.dump({"meta": {"generator": "tests/golden/make_oracle_n30.py", "numpy": np.__version__},
                   "cases": {name: rec}}, f, indent=0)
    print(f"wrote {out}: {name} n={w.num_qubits} G={w.num_gates} P={w.circuit.num_params} in {dt:.0f} s")


if __name__ == "__main__":
    main()
