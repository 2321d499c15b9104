"""Host-side cost breakdown of one gradient call (bind / native call / device)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time

import paper_2009_02823_b200 as sv
from paper_2009_02823_b200 import _native
from paper_2009_02823_b200.lowering import Problem

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = sv.build_workload(cfg)
inp = sv.BasisState(w.num_qubits)
eng = _native.engine(0)
for jit in (0, 1):
    eng.set_option("jit", jit)
    for _ in range(3):
        sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp)
    t0 = time.perf_counter()
    for _ in range(10):
        pr = Problem(w.circuit, w.theta, w.observable, inp, real_sums=True)
    t1 = time.perf_counter()
    st = {}
    for _ in range(10):
        sums, _, energy, stt = eng.reverse_sweep(pr.c, w.circuit.num_params, pr.num_derivs)
    t2 = time.perf_counter()
    print(f"jit={jit} bind {1e3*(t1-t0)/10:.3f} ms  native call {1e3*(t2-t1)/10:.3f} ms  device total {stt.ms_total:.3f} ms"
          f"  jit_passes {stt.jit_passes}  lower {stt.ms_host_lower:.3f} ms  prep {stt.ms_host_prep:.3f} ms")
