"""B200-native adjoint (reverse-mode) energy gradients -- drop-in for ``svgrad``'s gradient call.

    import paper_2009_02823_b200 as sv
    report = sv.reverse_mode_gradient(circuit, theta, observable, sv.init_basis_state(n))

Public names mirror the reference package root (svgrad/__init__.py:3-53) for
everything on the gradient path: circuit IR and factories, observables,
state containers, ``reverse_mode_gradient`` / ``non_hermitian_gradient`` and
the report types.  Reference ``svgrad`` objects are accepted as inputs too.
The engine is the CUDA library ``libsvgb200.so`` (sm_100a); there is no CPU
fallback -- without it the gradient calls raise ``NativeUnavailable``.
"""
from ._native import NativeUnavailable
from .adjoint import (
    GradientReport,
    LiveStateAudit,
    OpCounters,
    circuit_expectation,
    finite_difference_gradient,
    non_hermitian_gradient,
    reference_gradient,
    reverse_mode_gradient,
    sweep,
)
from . import distributed
from .configs import Workload, build_workload
from .ir import (
    Circuit,
    CustomParametric,
    FixedUnitary,
    Gate,
    NonInvertibleGateError,
    NonUnitary,
    PauliRotation,
    Phase,
    crx,
    cry,
    crz,
    cx,
    fixed,
    perturbed_derivative_scale,
    phase_gate,
    rp,
    rx,
    ry,
    rz,
)
from .operators import BUILTIN_OBSERVABLES, Observable, adjoint_observable, builtin_observable
from .state import BasisState, ShardSlice, StateVector, clone_state, init_basis_state, inner_product
from .textio import CircuitParseError, ObservableParseError, circuit_to_text, observable_to_text, parse_circuit, parse_observable

__version__ = "0.1.0"
