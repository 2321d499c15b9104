#!/usr/bin/env python3
"""The paper's Fig. 2 experiment on B200: gradient time vs circuit depth.

The paper times the O(P) reverse-mode schedule against an
O(P^2) one and fits log-log slopes (svgrad/bench.py:72-137 does the same on
CPU at N = 4-5).  Here: hardware-efficient layers (RY, RZ on every qubit + a
CNOT chain, the cfg 4 layer) at n qubits and L = 1..Lmax layers; each point is
the median of device-timed gradient calls (CUDA events on the engine stream).
The reverse sweep is timed at every depth; central differences over the GPU
expectation path (2P+1 forward sweeps, O(P^2) gate work) at the small depths.
A log-log fit of time vs P gives the scaling exponents.

    python tools/depth_sweep.py OUT.json [n] [Lmax]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_02823_b200 as sv
from paper_2009_02823_b200 import _native


def layers(n, L):
    gates, p = [], 0
    for _ in range(L):
        for q in range(n):
            gates.append(sv.ry(q, p))
            p += 1
        for q in range(n):
            gates.append(sv.rz(q, p))
            p += 1
        gates += [sv.cx(q, q + 1) for q in range(n - 1)]
    return sv.Circuit(n, tuple(gates), p)


def timed(fn, reps):
    stream = torch.cuda.current_stream()
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def fit(ps, ts):
    slope, icpt = np.polyfit(np.log(ps), np.log(ts), 1)
    return float(slope)


def main():
    out = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    lmax = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    eng = _native.engine(0)
    eng.set_stream(torch.cuda.current_stream().cuda_stream)
    obs = sv.Observable(n, tuple((1.0, "I" * i + "ZZ" + "I" * (n - i - 2)) for i in range(n - 1)) +
                        tuple((0.7, "I" * i + "X" + "I" * (n - i - 1)) for i in range(n)))
    inp = sv.BasisState(n)
    recs = []
    L = 1
    while L <= lmax:
        circ = layers(n, L)
        theta = np.random.default_rng([0, L]).uniform(0, 2 * np.pi, circ.num_params)
        rev = timed(lambda: sv.reverse_mode_gradient(circ, theta, obs, inp, engine=eng), 7)
        rec = {"layers": L, "params": circ.num_params, "gates": len(circ.gates), "reverse_ms": rev}
        if circ.num_params <= 2 * n * 8:
            rec["finite_difference_ms"] = timed(lambda: sv.finite_difference_gradient(circ, theta, obs, inp,
                                                                                      engine=eng), 1)
        recs.append(rec)
        print(json.dumps(rec), flush=True)
        L *= 2
    ps = [r["params"] for r in recs]
    summary = {"n": n, "points": recs,
               "reverse_loglog_slope": fit(ps[1:], [r["reverse_ms"] for r in recs[1:]]),
               "device": torch.cuda.get_device_name(0)}
    fd = [r for r in recs if "finite_difference_ms" in r]
    if len(fd) >= 3:
        summary["finite_difference_loglog_slope"] = fit([r["params"] for r in fd[1:]],
                                                        [r["finite_difference_ms"] for r in fd[1:]])
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "points"}))


if __name__ == "__main__":
    main()
