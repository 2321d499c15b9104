"""Shape of the engine's plan for a config without a GPU (nothing compiled):
passes, segments, layout changes, register ops, lane flips per sweep direction,
and the modelled reverse-sweep cost in register-op units."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_02823_b200 as sv  # noqa: E402
from paper_2009_02823_b200 import _native as N  # noqa: E402
from paper_2009_02823_b200.lowering import Problem  # noqa: E402


def stats(cfg, n, tile=0, reg_bits=0, low=0, max_gates=0, windows=1, shard_bits=0):
    lib = N.load()
    w = sv.build_workload(cfg, n)
    pr = Problem(w.circuit, w.theta, w.observable, sv.BasisState(w.num_qubits), real_sums=True)
    opts = (C.c_int64 * 6)(tile, reg_bits, low, max_gates, windows, shard_bits)
    out = (C.c_double * 16)()
    rc = lib.svg_debug_plan_stats(C.byref(pr.c), opts, out)
    if rc != 0:
        raise RuntimeError(lib.svg_last_error())
    keys = ("passes", "segments", "layout_changes", "reg_ops", "lane_flips", "max_slots", "lane_group_acc",
            "one_bit_exchanges")
    return {"fwd": dict(zip(keys, out[0:8])), "rev": dict(zip(keys, out[8:16])), "gates": len(w.circuit.gates)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--qubits", type=int, default=None)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--low", type=int, default=0)
    ap.add_argument("--max-gates", type=int, default=0)
    ap.add_argument("--windows", type=int, default=1)
    ap.add_argument("--shard-bits", type=int, default=0)
    a = ap.parse_args()
    print(stats(a.config, a.qubits, a.tile, 0, a.low, a.max_gates, a.windows, a.shard_bits))
