"""cProfile of repeated gradient calls (host-side Python overhead)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_02823_b200 as sv  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = sv.build_workload(cfg)
inp = sv.BasisState(w.num_qubits)
for _ in range(5):
    sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp)
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp, stats={})
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
