"""Circuit and observable text formats (the reference's file formats, restated).

Circuit text (svgrad/circuit.py:337-473): ``#`` starts a comment; the first
line is ``qubits <N>``, the second ``params <P>``, then one gate per line::

    rx q<t> p<k>   ry ...   rz ...      single-qubit rotations (alpha = -1/2)
    rp <axes> q<t1> [q<t2>] p<k>        Pauli-product rotation, axes over xyz
    phase q<t> p<k>
    h q<t>   x ...   y ...   z ...      fixed gates
    cx q<c> q<t>                        controlled X
    crx q<c> q<t> p<k>   cry ...   crz ...

Observable text (svgrad/observable.py:140-183): first line ``qubits <N>``,
then ``<re> <im> <factors>`` per term (factor string position j = qubit j).

Errors carry the 1-based line number exactly as the reference's
``CircuitParseError`` / ``ObservableParseError`` do ("line L: message").
Used by the CLI (cli.py) and for the configuration fixtures.
"""
from __future__ import annotations

from . import ir
from .operators import LETTERS, Observable


class CircuitParseError(ValueError):
    """Malformed circuit text; ``line`` is 1-based (0: whole file)."""

    def __init__(self, line: int, message: str):
        self.line = line
        super().__init__(f"line {line}: {message}")


class ObservableParseError(ValueError):
    def __init__(self, line: int, message: str):
        self.line = line
        super().__init__(f"line {line}: {message}")


_ROT = {"rx": "X", "ry": "Y", "rz": "Z"}
_CROT = {"crx": "X", "cry": "Y", "crz": "Z"}
_FIXED = ("h", "x", "y", "z")


def _lines(text: str):
    for lineno, raw in enumerate(text.splitlines(), start=1):
        body = raw.split("#", 1)[0].strip()
        if body:
            yield lineno, body.split()


def _header(tokens: list[str], keyword: str, line: int) -> int:
    if len(tokens) != 2 or tokens[0] != keyword or not tokens[1].isdigit():
        raise CircuitParseError(line, f"expected `{keyword} <n>`, got {' '.join(tokens)!r}")
    return int(tokens[1])


def _index(token: str, prefix: str, line: int, what: str, limit: int, table: str) -> int:
    if not token.startswith(prefix) or not token[len(prefix):].isdigit():
        raise CircuitParseError(line, f"expected {what} token like {prefix}3, got {token!r}")
    v = int(token[len(prefix):])
    if v >= limit:
        raise CircuitParseError(line, f"{what} {v} out of range ({table} has {limit})")
    return v


def parse_circuit(text: str) -> ir.Circuit:
    """Circuit text -> ``Circuit`` (this package's IR, reference field names)."""
    n = p = None
    gates = []
    for line, tok in _lines(text):
        if n is None:
            n = _header(tok, "qubits", line)
            if n < 1:
                raise CircuitParseError(line, "need at least one qubit")
            continue
        if p is None:
            p = _header(tok, "params", line)
            continue
        try:
            gates.append(_gate(tok, line, n, p))
        except CircuitParseError:
            raise
        except ValueError as exc:  # gate validation (e.g. repeated qubits)
            raise CircuitParseError(line, str(exc)) from exc
    if n is None or p is None:
        raise CircuitParseError(0, "missing `qubits`/`params` header lines")
    return ir.Circuit(n, tuple(gates), p)


def _gate(tok: list[str], line: int, n: int, p: int):
    def q(t):
        return _index(t, "q", line, "qubit", n, "circuit")

    def par(t):
        return _index(t, "p", line, "parameter", p, "table")

    def arity(count):
        if len(tok) != count:
            raise CircuitParseError(line, f"`{tok[0]}` takes {count - 1} argument(s)")

    op = tok[0]
    if op in _ROT:
        arity(3)
        return ir.Gate(ir.PauliRotation(_ROT[op]), (q(tok[1]),), (), (par(tok[2]),))
    if op == "rp":
        if len(tok) < 4:
            raise CircuitParseError(line, "`rp` takes axes, targets and a parameter")
        axes = tok[1]
        if any(a not in "xyz" for a in axes):
            raise CircuitParseError(line, f"axes must be over xyz, got {axes!r}")
        if not 1 <= len(axes) <= 2:
            raise CircuitParseError(line, "`rp` supports 1 or 2 targets")
        arity(3 + len(axes))
        return ir.Gate(ir.PauliRotation(axes.upper()), tuple(q(t) for t in tok[2:-1]), (), (par(tok[-1]),))
    if op == "phase":
        arity(3)
        return ir.Gate(ir.Phase(), (q(tok[1]),), (), (par(tok[2]),))
    if op in _FIXED:
        arity(2)
        return ir.fixed(op, q(tok[1]))
    if op == "cx":
        arity(3)
        return ir.cx(q(tok[1]), q(tok[2]))
    if op in _CROT:
        arity(4)
        return ir.Gate(ir.PauliRotation(_CROT[op]), (q(tok[2]),), (q(tok[1]),), (par(tok[3]),))
    raise CircuitParseError(line, f"unknown gate {op!r}")


def circuit_to_text(circuit) -> str:
    """Serialise; raises ValueError for gates the format cannot express."""
    out = [f"qubits {circuit.num_qubits}", f"params {circuit.num_params}"]
    for i, g in enumerate(circuit.gates):
        out.append(_gate_text(g, i))
    return "\n".join(out) + "\n"


def _gate_text(g, index: int) -> str:
    kind = ir.kind_name(g)
    ctrl = tuple(g.controls)
    if kind == "PauliRotation" and float(g.kind.alpha) == -0.5:
        axes = g.kind.axes.lower()
        if len(axes) == 1 and len(ctrl) == 1:
            return f"cr{axes} q{ctrl[0]} q{g.targets[0]} p{g.param_refs[0]}"
        if not ctrl:
            if len(axes) == 1:
                return f"r{axes} q{g.targets[0]} p{g.param_refs[0]}"
            return f"rp {axes} " + " ".join(f"q{t}" for t in g.targets) + f" p{g.param_refs[0]}"
    if kind == "Phase" and not ctrl:
        return f"phase q{g.targets[0]} p{g.param_refs[0]}"
    if kind == "FixedUnitary":
        name = getattr(g.kind, "name", None)
        if name in _FIXED and not ctrl:
            return f"{name} q{g.targets[0]}"
        if name == "x" and len(ctrl) == 1:
            return f"cx q{ctrl[0]} q{g.targets[0]}"
    raise ValueError(f"gate {index} ({kind}) is not representable in circuit text")


def parse_observable(text: str) -> Observable:
    n = None
    terms = []
    for line, tok in _lines(text):
        if n is None:
            if len(tok) != 2 or tok[0] != "qubits" or not tok[1].isdigit():
                raise ObservableParseError(line, f"expected `qubits <n>`, got {' '.join(tok)!r}")
            n = int(tok[1])
            continue
        if len(tok) != 3:
            raise ObservableParseError(line, "expected `<re> <im> <factors>`")
        try:
            coeff = complex(float(tok[0]), float(tok[1]))
        except ValueError as exc:
            raise ObservableParseError(line, f"bad coefficient: {exc}") from exc
        factors = tok[2]
        if len(factors) != n:
            raise ObservableParseError(line, f"factor string {factors!r} does not cover {n} qubits")
        if any(ch not in LETTERS for ch in factors):
            raise ObservableParseError(line, f"unknown factor letter in {factors!r}")
        terms.append((coeff, factors))
    if n is None:
        raise ObservableParseError(0, "missing `qubits` header line")
    if not terms:
        raise ObservableParseError(0, "observable has no terms")
    return Observable(n, tuple(terms))


def observable_to_text(obs) -> str:
    out = [f"qubits {obs.num_qubits}"]
    for c, f in obs.terms:
        c = complex(c)
        out.append(f"{c.real:.17g} {c.imag:.17g} {f}")
    return "\n".join(out) + "\n"
