#!/usr/bin/env python3
"""Gradient throughput and reverse-pass roofline vs qubits (BASELINE metric "... vs qubits").

Runs bench.py (one process per point: fresh engine, device-timed) for the layer
structure of each BASELINE config at several n and writes one JSON record per
point plus a markdown table.

    python tools/qubit_sweep.py OUT.json [cfg:n,n,...] ...
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(cfg, n):
    steps = 20 if n <= 22 else (5 if n <= 26 else 2)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(cfg), "--qubits", str(n), "--steps",
           str(steps), "--warmup", "3", "--no-cpu-baseline", "--no-e2e"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    S = 16 << n
    return {
        "cfg": cfg, "n": n, "gates": line["config"]["num_gates"], "grad_per_s": line["value"],
        "ms_per_step": line["ms_per_step"], "phase_ms": line["phase_ms"], "passes": line["passes"],
        "rev_roofline_frac": line["roofline"]["frac"], "rev_achieved_gbs": line["roofline"]["achieved"],
        "effective_gate_level_gbs": line["effective_gate_level_gbs"], "state_bytes": S,
        "rev_fp64_frac": (line.get("roofline_fp64") or {}).get("frac"),
        "clocks": line["clocks"],
    }


def main():
    out_path = sys.argv[1]
    specs = sys.argv[2:] or ["2:14,16,18,20,22,24,26,28", "3:20,22,24,26,28", "4:24,26,28,30", "5:24,26,28,30"]
    recs = []
    for spec in specs:
        cfg, ns = spec.split(":")
        for n in ns.split(","):
            try:
                recs.append(run(int(cfg), int(n)))
                r = recs[-1]
                print(f"cfg{cfg} n={n}: {r['grad_per_s']:.4g} grad/s, {r['ms_per_step']:.4g} ms, "
                      f"reverse pass {r['rev_achieved_gbs']:.0f} GB/s ({r['rev_roofline_frac']:.2f})", flush=True)
            except Exception as exc:  # keep sweeping
                print(f"cfg{cfg} n={n}: failed: {exc}", flush=True)
    with open(out_path, "w") as f:
        json.dump(recs, f, indent=1)


if __name__ == "__main__":
    main()
