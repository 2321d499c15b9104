"""ctypes binding of libsvgb200.so (the C-ABI in include/svgrad_b200.h).

The product path has no fallback: if the library or a CUDA device is missing,
every call raises ``NativeUnavailable`` -- there is no CPU implementation
behind these entry points.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsvgb200.so")
ABI_VERSION = 3

SVG_OK, SVG_EINVAL, SVG_ENOMEM, SVG_ECUDA, SVG_ENCCL, SVG_EUNSUPPORTED = range(6)
FORM_PAULI, FORM_MAT = 0, 1

EXPORTED = (
    "svg_abi_version", "svg_last_error", "svg_device_count", "svg_engine_create",
    "svg_engine_destroy", "svg_engine_set_stream", "svg_engine_set_option",
    "svg_reverse_sweep", "svg_expectation", "svg_plan_inspect", "svg_engine_create_virtual",
    "svg_nccl_unique_id", "svg_engine_create_sharded", "svg_plan_schedule",
)


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a device) is not available; there is no fallback."""


class c128(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


C128x16 = c128 * 16


class svg_gate(C.Structure):
    _fields_ = [
        ("form", C.c_int32), ("ntargets", C.c_int32), ("targets", C.c_int32 * 2),
        ("ctrl_mask", C.c_uint64), ("x_mask", C.c_uint64), ("z_mask", C.c_uint64),
        ("n_y", C.c_int32), ("nderiv", C.c_int32),
        ("fwd", C128x16), ("rewind", C128x16), ("adjoint", C128x16),
    ]


class svg_deriv(C.Structure):
    _fields_ = [
        ("gate", C.c_int32), ("param_ref", C.c_int32), ("form", C.c_int32),
        ("basis", C.c_int32), ("k", C128x16),
    ]


class svg_pauli_term(C.Structure):
    _fields_ = [
        ("coeff", c128), ("x_mask", C.c_uint64), ("z_mask", C.c_uint64),
        ("n_y", C.c_int32), ("reserved", C.c_int32),
    ]


class svg_product_term(C.Structure):
    _fields_ = [("coeff", c128), ("first_factor", C.c_int32), ("num_factors", C.c_int32)]


class svg_factor(C.Structure):
    _fields_ = [("qubit", C.c_int32), ("reserved", C.c_int32), ("m", c128 * 4)]


class svg_problem(C.Structure):
    _fields_ = [
        ("num_qubits", C.c_int32), ("num_params", C.c_int32), ("num_gates", C.c_int32),
        ("num_derivs", C.c_int32), ("num_terms", C.c_int32), ("flags", C.c_int32),
        # table pointers held as addresses (c_void_p): assigning a numpy array's
        # .ctypes.data is ~10x cheaper per call than data_as(POINTER(...))
        ("gates", C.c_void_p), ("derivs", C.c_void_p),
        ("terms", C.c_void_p), ("input_basis", C.c_int64),
        ("input_amps", C.c_void_p),
        ("num_product_terms", C.c_int32), ("num_factors", C.c_int32),
        ("product_terms", C.c_void_p), ("factors", C.c_void_p),
    ]


class svg_stats(C.Structure):
    _fields_ = [
        ("ms_total", C.c_double), ("ms_forward", C.c_double), ("ms_observable", C.c_double),
        ("ms_reverse", C.c_double), ("ms_other", C.c_double), ("launches", C.c_int64),
        ("fwd_passes", C.c_int32), ("obs_passes", C.c_int32), ("rev_passes", C.c_int32),
        ("tile_qubits", C.c_int32), ("pass_bytes", C.c_int64), ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64), ("segments", C.c_int32), ("reg_bits", C.c_int32),
        ("swaps", C.c_int32), ("jit_passes", C.c_int32), ("exchange_bytes", C.c_int64),
        ("ms_host_lower", C.c_double), ("ms_host_prep", C.c_double), ("nonfinite", C.c_int32),
        ("reserved", C.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None
_lib_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load and type the library once; raises NativeUnavailable if absent."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -m paper_2009_02823_b200._build` "
                "(there is no CPU fallback for the gradient engine)"
            )
        lib = C.CDLL(path)
        lib.svg_abi_version.restype = C.c_int
        lib.svg_last_error.restype = C.c_char_p
        lib.svg_device_count.argtypes = [C.POINTER(C.c_int)]
        lib.svg_engine_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        lib.svg_engine_destroy.argtypes = [C.c_void_p]
        lib.svg_engine_set_stream.argtypes = [C.c_void_p, C.c_void_p]
        lib.svg_engine_set_option.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        lib.svg_reverse_sweep.argtypes = [  # sums / derivs: complex128 buffers (numpy-owned)
            C.c_void_p, C.POINTER(svg_problem), C.c_void_p, C.c_void_p,
            C.POINTER(c128), C.POINTER(svg_stats),
        ]
        lib.svg_expectation.argtypes = [C.c_void_p, C.POINTER(svg_problem), C.POINTER(c128), C.POINTER(svg_stats)]
        lib.svg_plan_inspect.argtypes = [
            C.POINTER(svg_problem), C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
            C.POINTER(C.c_int32), C.POINTER(C.c_int32),
        ]
        lib.svg_plan_schedule.argtypes = [
            C.POINTER(svg_problem), C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
            C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
        ]
        lib.svg_engine_create_virtual.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        lib.svg_nccl_unique_id.argtypes = [C.c_void_p]
        lib.svg_engine_create_sharded.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
        for name in EXPORTED:
            getattr(lib, name).restype = C.c_char_p if name == "svg_last_error" else C.c_int
        if lib.svg_abi_version() != ABI_VERSION:
            raise NativeUnavailable(f"ABI mismatch: library {lib.svg_abi_version()}, wrapper {ABI_VERSION}")
        _lib = lib
        return lib


def check(code: int) -> None:
    """Map a C-ABI status onto the reference's exception types."""
    if code == SVG_OK:
        return
    msg = (_lib.svg_last_error() or b"").decode(errors="replace")
    if code == SVG_EINVAL:
        raise ValueError(msg)
    if code == SVG_ENOMEM:
        raise MemoryError(msg)
    if code == SVG_EUNSUPPORTED:
        raise NativeUnavailable(msg)
    raise RuntimeError(f"svgrad_b200 native error {code}: {msg}")


class Engine:
    """One device context: streams, cached HBM buffers, kernel attributes.

    Not re-entrant (the reference's single-writer contract, pkg/README.md:71-73):
    calls on one Engine are serialised by a lock; ctypes releases the GIL
    for the duration of the native call.
    """

    def __init__(self, device: int = 0, *, shards: int = 1, rank: int | None = None,
                 nccl_id: bytes | None = None):
        """shards == 1: one device, whole state.  shards > 1 and rank None: virtual
        shards on this device.  rank given: one rank of a `shards`-GPU NCCL job."""
        self.lib = load()
        handle = C.c_void_p()
        if shards == 1 and rank is None:
            check(self.lib.svg_engine_create(int(device), C.byref(handle)))
        elif rank is None:
            check(self.lib.svg_engine_create_virtual(int(device), int(shards), C.byref(handle)))
        else:
            buf = C.create_string_buffer(bytes(nccl_id or b""), 128)
            check(self.lib.svg_engine_create_sharded(int(device), int(shards), int(rank), buf, C.byref(handle)))
        self.handle = handle
        self.device = device
        self.shards = shards
        self.rank = rank
        self.lock = threading.Lock()

    def set_option(self, key: str, value: int) -> None:
        check(self.lib.svg_engine_set_option(self.handle, key.encode(), int(value)))

    def set_stream(self, stream_ptr: int | None) -> None:
        check(self.lib.svg_engine_set_stream(self.handle, C.c_void_p(stream_ptr or None)))

    def reverse_sweep(self, problem: svg_problem, num_params: int, num_derivs: int):
        """(sums complex128[P], derivs complex128[D], energy, stats) of one sweep."""
        import numpy as np

        sums = np.zeros(max(1, num_params), dtype=np.complex128)
        derivs = np.zeros(max(1, num_derivs), dtype=np.complex128)
        energy = c128()
        stats = svg_stats()
        with self.lock:
            check(self.lib.svg_reverse_sweep(self.handle, C.byref(problem), sums.ctypes.data, derivs.ctypes.data,
                                             C.byref(energy), C.byref(stats)))
        return sums[:num_params], derivs[:num_derivs], energy, stats

    def expectation(self, problem: svg_problem):
        energy = c128()
        stats = svg_stats()
        with self.lock:
            check(self.lib.svg_expectation(self.handle, C.byref(problem), C.byref(energy), C.byref(stats)))
        return energy, stats

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.svg_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def plan_inspect(problem: svg_problem, tile_qubits: int = 0, sms: int = 0):
    """Planner output without a GPU: (order, pass_start, qmasks, tile_qubits)."""
    import numpy as np

    lib = load()
    G = max(1, problem.num_gates)
    order = np.zeros(G, dtype=np.int32)
    start = np.zeros(G + 1, dtype=np.int32)
    qmask = np.zeros(G, dtype=np.uint64)
    npasses, k = C.c_int32(), C.c_int32()
    check(lib.svg_plan_inspect(C.byref(problem), int(tile_qubits), int(sms), order.ctypes.data,
                               start.ctypes.data, qmask.ctypes.data, C.byref(npasses), C.byref(k)))
    m = npasses.value
    return order[: problem.num_gates], start[: m + 1], qmask[:m], k.value


def nccl_unique_id() -> bytes:
    lib = load()
    buf = C.create_string_buffer(128)
    check(lib.svg_nccl_unique_id(buf))
    return buf.raw


def plan_schedule(problem: svg_problem, shards: int, tile_qubits: int = 0, sms: int = 0):
    """Sharded schedule without a GPU: list of ('pass', gate_indices, qmask) / ('swap', gbit, lpos)."""
    import numpy as np

    lib = load()
    G = max(1, problem.num_gates)
    cap = G * (2 * max(1, shards).bit_length() + 3) + 8
    order = np.zeros(G, dtype=np.int32)
    start = np.zeros(cap + 1, dtype=np.int32)
    swap = np.zeros(cap, dtype=np.int32)
    qmask = np.zeros(cap, dtype=np.uint64)
    nsteps, k = C.c_int32(), C.c_int32()
    check(lib.svg_plan_schedule(C.byref(problem), int(shards), int(tile_qubits), int(sms), order.ctypes.data,
                                start.ctypes.data, swap.ctypes.data, qmask.ctypes.data, C.byref(nsteps),
                                C.byref(k)))
    steps = []
    for j in range(nsteps.value):
        if swap[j]:
            code = int(swap[j]) - 1
            steps.append(("swap", code >> 8, code & 0xFF))
        else:
            steps.append(("pass", order[start[j]:start[j + 1]].tolist(), int(qmask[j])))
    return steps, k.value


_engines: dict[int, Engine] = {}


def engine(device: int = 0) -> Engine:
    """Process-wide engine per device (created on first use)."""
    e = _engines.get(device)
    if e is None:
        e = _engines[device] = Engine(device)
    return e
