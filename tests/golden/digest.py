"""Structural digests of a workload (fixtures record them; tests recompute them)."""
import hashlib


def circuit_digest(circuit) -> str:
    """Structure-only digest: kind class name, targets, controls, refs per gate."""
    h = hashlib.sha256()
    h.update(f"{circuit.num_qubits}/{circuit.num_params}".encode())
    for g in circuit.gates:
        kind = g.kind
        extra = getattr(kind, "axes", "") + str(getattr(kind, "alpha", ""))
        h.update(f"|{type(kind).__name__}:{extra}:{g.targets}:{g.controls}:{g.param_refs}".encode())
    return h.hexdigest()[:16]


def obs_digest(obs) -> str:
    h = hashlib.sha256()
    for c, f in obs.terms:
        h.update(f"{complex(c)!r}:{f};".encode())
    return h.hexdigest()[:16]
