"""Generate golden gradient fixtures by running the REFERENCE implementation.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src; nothing on the GPU box reads it):

    python tests/golden/make_golden.py                 # small + config cases -> golden_small.json
    python tests/golden/make_golden.py --large cfg2     # one large case -> golden_cfg2.json

Each record holds the reference's ``reverse_mode_gradient`` output (or
``non_hermitian_gradient`` for non-Hermitian cases): values, energy and the
exact OpCounters, plus ``reference_gradient`` values for small cases as a
second pin.  Circuits are rebuilt in the tests from ``tests/cases.py``; a
structural digest of the circuit and a checksum of theta/input are stored so
a drifting builder is caught.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))             # tests/
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))  # repo root
REFERENCE_SRC = "/root/reference/pkg/src"

from digest import circuit_digest, obs_digest  # noqa: E402


def cplx(a):
    a = np.asarray(a, dtype=complex).ravel()
    return [[float(z.real), float(z.imag)] for z in a]


def run_case(sv, name, build, with_reference_engine):
    from cases import input_state

    spec = build(sv)
    circ, theta, obs = spec["circuit"], spec["theta"], spec["obs"]
    inp = input_state(sv, circ.num_qubits, spec["input"])
    t0 = time.perf_counter()
    if spec["method"] == "non_hermitian":
        rep = sv.non_hermitian_gradient(circ, theta, obs, inp)
    else:
        rep = sv.reverse_mode_gradient(circ, theta, obs, inp)
    dt = time.perf_counter() - t0
    rec = {
        "method": spec["method"],
        "num_qubits": circ.num_qubits,
        "num_gates": len(circ.gates),
        "num_params": circ.num_params,
        "circuit_digest": circuit_digest(circ),
        "obs_digest": obs_digest(obs),
        "theta_sum": float(np.sum(theta)),
        "input": list(spec["input"]),
        "input_norm2": float(np.vdot(inp.amplitudes, inp.amplitudes).real),
        "values": cplx(rep.values),
        "energy": cplx([rep.energy])[0],
        "counters": vars(rep.counters),
        "reference_seconds": dt,
    }
    if with_reference_engine and spec["method"] == "reverse":
        rec["reference_gradient_values"] = cplx(sv.reference_gradient(circ, theta, obs, inp).values)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", default=None, help="name of one large_config_cases() entry")
    args = ap.parse_args()
    sys.path.insert(0, REFERENCE_SRC)
    import svgrad as sv
    import cases

    if args.large:
        recs = {args.large: run_case(sv, args.large, cases.large_config_cases()[args.large], False)}
        out = os.path.join(HERE, f"golden_{args.large}.json")
    else:
        recs = {}
        table = dict(cases.small_cases())
        table.update(cases.config_cases())
        for name, build in table.items():
            recs[name] = run_case(sv, name, build, with_reference_engine=True)
        out = os.path.join(HERE, "golden_small.json")
    meta = {
        "generator": "tests/golden/make_golden.py",
        "reference": "svgrad 0.1.0 from /root/reference/pkg/src (imported in place)",
        "numpy": np.__version__,
    }
    with open(out, "w") as f:
        json.dump({"meta": meta, "cases": recs}, f, indent=0)
    print(f"wrote {out}: {len(recs)} cases")


if __name__ == "__main__":
    main()
