"""Golden fixtures for the text formats and the CLI, produced by the REFERENCE.

Run in the build container only (imports the read-only reference from
/root/reference/pkg/src; nothing on the GPU box reads it):

    python tests/golden/make_textio_golden.py   -> tests/golden/golden_textio.json

Records: the reference's ``circuit_to_text`` / ``observable_to_text`` of the
configuration circuits (cfg 1-5 at reduced size, built with the reference's
own factories through ``configs.py``), the ``str()`` of the parse error the
reference raises for each malformed input below, and its CLI report for a
few small files (stdout text and exit code).
"""
from __future__ import annotations

import contextlib
import io
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))  # repo root
sys.path.insert(0, "/root/reference/pkg/src")

BAD_CIRCUITS = [
    "qubits 2\nparams 1\nrw q0 p0\n",
    "qubits 2\nparams 1\nrx q2 p0\n",
    "qubits 2\nparams 1\nrx q0 p1\n",
    "qubits 2\nparams 1\nrx q0\n",
    "qubits 2\nparams 1\nrx x0 p0\n",
    "qubits two\nparams 1\n",
    "qubits 2\n",
    "qubits 0\nparams 0\n",
    "qubits 3\nparams 1\nrp xyz q0 q1 q2 p0\n",
    "qubits 3\nparams 1\nrp xa q0 q1 p0\n",
    "qubits 3\nparams 1\nrp xx q0 q1\n",
    "# comment only\n\nqubits 2 # trailing\nparams 1\ncx q0 q0\n",
    "qubits 2\nparams 1\ncry q0 q1\n",
    "qubits 2\nparams 1\nh q0 q1\n",
]
BAD_OBSERVABLES = [
    "qubits 2\n1.0 0.0 ZZZ\n",
    "qubits 2\n1.0 ZZ\n",
    "qubits 2\n1.0 0.0 ZQ\n",
    "qubits 2\n1.0 x ZZ\n",
    "qubits 2\n",
    "1.0 0.0 ZZ\n",
]
CLI_CASES = [
    ("qubits 1\nparams 1\nry q0 p0\n", "z_all", "1.5707963267948966", "reverse"),
    ("qubits 1\nparams 1\nry q0 p0\n", "z_all", "0.3", "reverse"),
    ("qubits 3\nparams 4\nrx q0 p0\nry q1 p1\ncx q0 q2\ncrz q1 q2 p2\nphase q0 p3\nrz q2 p1\n", "hadamard_all",
     "0.3,1.2,-0.7,2.2", "reverse"),
    ("qubits 2\nparams 2\nry q0 p0\nrp zx q0 q1 p1\nh q1\n", "obs:qubits 2\n0.5 0.0 XZ\n0.0 0.7 +Y\n", "0.4,-1.1",
     "reverse"),
    ("qubits 2\nparams 1\nry q3 p0\n", "z_all", "0.1", "reverse"),
    # the O(P^2) reference schedule (svgrad/cli.py:79-89): counters G + A(G-1) / A+1 clones
    ("qubits 1\nparams 1\nry q0 p0\n", "z_all", "0.3", "reference"),
    ("qubits 3\nparams 4\nrx q0 p0\nry q1 p1\ncx q0 q2\ncrz q1 q2 p2\nphase q0 p3\nrz q2 p1\n", "hadamard_all",
     "0.3,1.2,-0.7,2.2", "reference"),
    ("qubits 3\nparams 3\nry q0 p0\ncry q0 q1 p1\nrp xy q1 q2 p2\nh q2\n", "hadamard_all", "0.9,-0.4,1.7", "reference"),
    ("qubits 2\nparams 2\nry q0 p0\nrp zx q0 q1 p1\nh q1\n", "obs:qubits 2\n0.5 0.0 XZ\n0.0 0.7 +Y\n", "0.4,-1.1",
     "reference"),
]


def main():
    import svgrad
    from svgrad import cli as rcli
    from svgrad.circuit import circuit_to_text, parse_circuit
    from svgrad.observable import observable_to_text, parse_observable

    from paper_2009_02823_b200 import configs

    api = configs.SimpleNamespace(Circuit=svgrad.Circuit, Observable=svgrad.Observable, rx=svgrad.rx,
                                  ry=svgrad.ry, rz=svgrad.rz, cx=svgrad.cx, cry=svgrad.cry, rp=svgrad.rp)
    out = {"config_text": {}, "bad_circuits": [], "bad_observables": [], "cli": []}
    for cfg, n in ((1, 10), (2, 8), (3, 8), (4, 8), (5, 8)):
        w = configs.build_workload(cfg, n, api=api)
        out["config_text"][f"cfg{cfg}_n{n}"] = {"circuit": circuit_to_text(w.circuit),
                                               "observable": observable_to_text(w.observable)}
    for text in BAD_CIRCUITS:
        try:
            parse_circuit(text)
            out["bad_circuits"].append([text, None])
        except ValueError as exc:
            out["bad_circuits"].append([text, str(exc)])
    for text in BAD_OBSERVABLES:
        try:
            parse_observable(text)
            out["bad_observables"].append([text, None])
        except ValueError as exc:
            out["bad_observables"].append([text, str(exc)])
    with tempfile.TemporaryDirectory() as tmp:
        for circ, obs, params, method in CLI_CASES:
            cpath = os.path.join(tmp, "c.circ")
            with open(cpath, "w") as f:
                f.write(circ)
            ospec = obs
            if obs.startswith("obs:"):
                ospec = os.path.join(tmp, "o.obs")
                with open(ospec, "w") as f:
                    f.write(obs[4:])
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(io.StringIO()):
                code = rcli.main(["grad", cpath, ospec, params, "--method", method])
            out["cli"].append({"circuit": circ, "observable": obs, "params": params, "method": method,
                               "exit_code": code, "stdout": buf.getvalue()})
    with open(os.path.join(HERE, "golden_textio.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote golden_textio.json")


if __name__ == "__main__":
    main()
