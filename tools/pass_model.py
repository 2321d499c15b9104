#!/usr/bin/env python3
"""Reverse-pass cost model on the GPU: synthetic circuits whose passes hold g
rotations of one kind, timed per pass (phase_ms / passes) for several g.
A linear fit t_pass = t0 + g * t_gate separates the per-pass memory cost from
the per-gate compute cost.

    python tools/pass_model.py [n]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_02823_b200 as sv
from paper_2009_02823_b200 import _native, ir, operators

n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = _native.engine(0)
stream = torch.cuda.current_stream()
eng.set_stream(stream.cuda_stream)
for kv in os.environ.get("SVGB_OPTS", "").split():  # extra engine options KEY=VALUE
    k_, v_ = kv.split("=")
    eng.set_option(k_, int(v_))
obs = operators.Observable(n, ((1.0, "Z" + "I" * (n - 1)),))
basis = sv.BasisState(n)

FAMILIES = {
    "ry_reg": lambda L: [ir.ry(5 + (i % 4), i) for i in range(L)],             # register flips, one segment
    "rx_reg": lambda L: [ir.rx(5 + (i % 4), i) for i in range(L)],
    "ry_lane": lambda L: [ir.ry(i % 4, i) for i in range(L)],                  # lane flips (shuffles)
    "rz": lambda L: [ir.rz(5 + (i % 4), i) for i in range(L)],                 # diagonal (fused runs)
    "ry_2seg": lambda L: [ir.ry(5 + (i % 6), i) for i in range(L)],            # 6 non-lane qubits: 2 segments
    "cry_reg": lambda L: [ir.cry(5 + (i % 4), 5 + ((i + 1) % 4), i) for i in range(L)],
}
res = {}
fams = sys.argv[3].split(",") if len(sys.argv) > 3 else list(FAMILIES)
gs = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [4, 8, 16, 32]
for fam in fams:
    mk = FAMILIES[fam]
    for g in gs:
        L = 8 * g
        gates = mk(L)
        circ = ir.Circuit(n, tuple(gates), L)
        theta = np.random.default_rng(1).uniform(0, 2 * np.pi, L)
        eng.set_option("max_gates_per_pass", g)
        st = {}
        for _ in range(2):
            sv.reverse_mode_gradient(circ, theta, obs, basis, stats=st, engine=eng)
        ts = []
        for _ in range(3):
            st = {}
            sv.reverse_mode_gradient(circ, theta, obs, basis, stats=st, engine=eng)
            ts.append((st["ms_reverse"] / st["rev_passes"], st["ms_forward"] / st["fwd_passes"], st["rev_passes"]))
        rev = min(t[0] for t in ts) * 8
        fwd = min(t[1] for t in ts) * 8
        npass = ts[0][2]
        res[f"{fam}_{g}"] = {"gates_per_pass": g, "rev_ms_per_pass": rev / 8, "fwd_ms_per_pass": fwd / 8}
        print(fam, g, npass, f"rev/pass {rev / 8:.3f} ms fwd/pass {fwd / 8:.3f} ms", flush=True)
json.dump(res, open(sys.argv[2] if len(sys.argv) > 2 else "/dev/null", "w"), indent=1)
