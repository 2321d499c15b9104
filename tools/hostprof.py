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

# per-phase host time of lower() (svg_debug_phase_ms), jit on
import ctypes as C
lib = _native.load()
eng.set_option("jit", 1)
out = (C.c_double * 9)()
lib.svg_debug_phase_ms(out, 1)
reps = 20
t0 = time.perf_counter()
for _ in range(reps):
    sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp)
t1 = time.perf_counter()
lib.svg_debug_phase_ms(out, 1)
names = ["schedule+gates", "generators", "segments", "forward emit", "observable emit", "reverse emit",
         "sizing", "jit lookup", "-"]
print(f"API call wall {1e3 * (t1 - t0) / reps:.3f} ms; lower() phases (ms/call): " +
      ", ".join(f"{n} {out[i] / reps:.4f}" for i, n in enumerate(names[:8])))
