/*
 * svgrad_b200.h -- C-ABI of the B200 adjoint-gradient engine (libsvgb200.so).
 *
 * Drop-in boundary for the reference's gradient call.  The reference
 * (pure Python, no FFI) exposes the hot path as
 *     svgrad.reverse_mode_gradient(circuit, params, obs, input_state, audit)
 *       -> GradientReport                        (svgrad/gradients.py:176-198)
 * built on the internal seam
 *     _reverse_sweep(circuit, params, obs, input_state, counters, audit)
 *       -> (sums complex[P], energy complex)     (svgrad/gradients.py:128-173)
 * which non_hermitian_gradient (svgrad/gradients.py:240-259) also calls.
 * svg_reverse_sweep() below replaces _reverse_sweep one-for-one: it returns
 * the COMPLEX per-parameter sums (callers form 2*Re for Hermitian operators,
 * or conj(sums_A) + sums_Adag for non-Hermitian ones) and the energy.
 *
 * Everything crossing this boundary is plain C: host pointers, sizes and
 * status codes; no torch or CUDA types.  Binding theta to matrices, inverse
 * computation (NonInvertibleGateError) and argument validation stay on the
 * host side, before the call, exactly where the reference does them
 * (svgrad/gradients.py:92-125), so error types and messages are unchanged.
 *
 * Conventions (reference Appendix A of SURVEY.md):
 *   - amplitudes are complex128, little-endian: qubit q is bit q of the index
 *     (svgrad/statevector.py:3-4);
 *   - 2-target matrices use sub-index bit k <-> targets[k]
 *     (svgrad/statevector.py:100-104);
 *   - a gate acts only where every control bit is 1 (svgrad/statevector.py:97-98).
 */
#ifndef SVGRAD_B200_H
#define SVGRAD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVG_ABI_VERSION 3
#define SVG_MAX_QUBITS 40

typedef struct { double re, im; } svg_c128;

/* status codes */
enum {
  SVG_OK = 0,
  SVG_EINVAL = 1,       /* invalid argument  -> ValueError   */
  SVG_ENOMEM = 2,       /* device allocation -> MemoryError  */
  SVG_ECUDA = 3,        /* CUDA runtime error -> RuntimeError */
  SVG_ENCCL = 4,        /* NCCL error         -> RuntimeError */
  SVG_EUNSUPPORTED = 5  /* e.g. no CUDA device -> RuntimeError */
};

/* gate / generator forms */
enum {
  SVG_FORM_PAULI = 0, /* op = c[0]*I + c[1]*P, P the Pauli product given by x/z/n_y */
  SVG_FORM_MAT = 1    /* op = dense 2^k x 2^k matrix (row-major) on targets */
};

/* One circuit gate, bound to theta on the host.
 * Replaces: gate_matrix / _bind / _rewind_matrices (svgrad/circuit.py:228-243,
 * svgrad/gradients.py:109-125).  For SVG_FORM_PAULI the three operators share
 * the gate's Pauli product P = prod_t sigma_{axis_t} (x_mask: X or Y on the
 * qubit; z_mask: Z or Y; n_y: number of Y factors), and only c[0], c[1] of
 * each array are read.  For SVG_FORM_MAT the arrays hold 2x2 (first 4) or
 * 4x4 (all 16) row-major matrices. */
typedef struct {
  int32_t form;
  int32_t ntargets;     /* 1 or 2 */
  int32_t targets[2];
  uint64_t ctrl_mask;   /* controls: bit q set => qubit q must be 1 */
  uint64_t x_mask;      /* PAULI only */
  uint64_t z_mask;      /* PAULI only */
  int32_t n_y;          /* PAULI only */
  int32_t nderiv;       /* number of local parameters (arity) */
  svg_c128 fwd[16];     /* U: forward pass (svgrad/gradients.py:149-150)        */
  svg_c128 rewind[16];  /* U^-1 on phi: adjoint, or inverse for NonUnitary (:160) */
  svg_c128 adjoint[16]; /* U^dagger on lambda (:167-168)                         */
} svg_gate;

/* Derivative generator of one (gate, local parameter) occurrence.
 * Contribution to sums[param_ref] is <lambda_i | K | phi_i>, phi_i the state
 * BEFORE gate i and lambda_i = U_{i+1}^dag..U_G^dag H psi.  K folds in the
 * deferred scalar and the control projector of apply_gate_derivative
 * (svgrad/circuit.py:302-334) and the sums += scalar*<bra|probe> of
 * svgrad/gradients.py:161-165.  PAULI form shares the gate's P. */
typedef struct {
  int32_t gate;
  int32_t param_ref;
  int32_t form;
  int32_t basis;        /* 0: K acts on phi_i (before gate i, the reference's probe order);
                           1: K acts on phi_{i+1} (after gate i); the engine converts via
                           K_post = K_pre * U^-1 / K_pre = K_post * U */
  svg_c128 k[16];
} svg_deriv;

/* One Pauli string of the observable (terms with few H,+,- letters pre-expanded
 * on the host; wider ones go to svg_product_term).
 * Replaces the per-term loop of apply_observable (svgrad/observable.py:79-100). */
typedef struct {
  svg_c128 coeff;
  uint64_t x_mask;
  uint64_t z_mask;
  int32_t n_y;
  int32_t reserved;
} svg_pauli_term;

/* One product term coeff * (x)_q F_q of the observable with arbitrary 2x2
 * factors F_q (row-major, on distinct qubits): the letters H, + and - (and any
 * Pauli letters of the same term) as matrices, applied factor by factor --
 * Walsh-Hadamard butterflies for H -- instead of an expansion into 2^w Pauli
 * strings (hadamard_all = 2^N strings; svgrad/observable.py:19-27,79-100,
 * svgrad/bench.py:94).  factors[first_factor .. first_factor + num_factors). */
typedef struct {
  svg_c128 coeff;
  int32_t first_factor;
  int32_t num_factors;
} svg_product_term;

typedef struct {
  int32_t qubit;
  int32_t reserved;
  svg_c128 m[4];
} svg_factor;

/* svg_problem.flags */
#define SVG_FLAG_REAL_SUMS 1  /* only Re(sums) is needed (Hermitian 2*Re path); imag may be 0 */
#define SVG_FLAG_INPUT_LOCAL 2 /* input_amps holds only this engine's amplitudes: on an NCCL rank the
                                  2^(n - log2 world) amplitudes of its shard (indices rank * 2^(n - log2
                                  world) ...), elsewhere the whole state; no per-rank 2^n host array */

typedef struct {
  int32_t num_qubits;
  int32_t num_params;
  int32_t num_gates;
  int32_t num_derivs;        /* = sum of arities, gate-major order */
  int32_t num_terms;
  int32_t flags;             /* SVG_FLAG_* */
  const svg_gate* gates;
  const svg_deriv* derivs;
  const svg_pauli_term* terms;
  int64_t input_basis;       /* |input_basis> when input_amps == NULL */
  const svg_c128* input_amps;/* host array of 2^n amplitudes, or NULL */
  /* ABI 2: product terms (applied after the Pauli strings; the observable is the sum of both) */
  int32_t num_product_terms;
  int32_t num_factors;
  const svg_product_term* product_terms;
  const svg_factor* factors;
} svg_problem;

typedef struct {
  double ms_total;           /* device time of the whole sweep (CUDA events) */
  double ms_forward;
  double ms_observable;
  double ms_reverse;
  double ms_other;           /* init/upload/finalize/download */
  int64_t launches;          /* kernels launched by this call */
  int32_t fwd_passes;
  int32_t obs_passes;
  int32_t rev_passes;
  int32_t tile_qubits;
  int64_t pass_bytes;        /* HBM state bytes the passes must move (read+write) */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int32_t segments;          /* register-tile segments over all passes (0: shared-memory kernels) */
  int32_t reg_bits;          /* amplitudes per thread per buffer = 2^reg_bits (register kernels) */
  int32_t swaps;             /* sharded engines: qubit swaps (rank bit <-> local qubit) per sweep */
  int32_t jit_passes;        /* register-tile launches run by circuit-specialised (NVRTC) kernels */
  int64_t exchange_bytes;    /* sharded engines: bytes one shard sends to partners per sweep */
  double ms_host_lower;      /* host time: validation + lowering (plans, op tables, kernel lookup) */
  double ms_host_prep;       /* host time: staging buffers between lowering and the first launch */
  /* ABI 3: numeric guard -- device sums (per-shard finalized partials of every
   * derivative slot and the energy) that came out NaN or infinite */
  int32_t nonfinite;
  int32_t reserved;
} svg_stats;

typedef struct svg_engine svg_engine;

int svg_abi_version(void);
const char* svg_last_error(void);   /* thread-local message of the last failure */
int svg_device_count(int* out);

int svg_engine_create(int device, svg_engine** out);
/* Sharded engines: the state is split over `shards` (a power of two) by its
 * top log2(shards) qubits.  A virtual engine holds every shard on one device
 * (exercises the distributed schedule on one GPU); an NCCL engine is one rank
 * of a one-process-per-GPU job (all ranks call it with the same unique id,
 * from svg_nccl_unique_id on rank 0).  Results are complete on every rank. */
int svg_engine_create_virtual(int device, int shards, svg_engine** out);
int svg_nccl_unique_id(uint8_t id_out[128]);
int svg_engine_create_sharded(int device, int world, int rank, const uint8_t nccl_id[128], svg_engine** out);
int svg_engine_destroy(svg_engine* e);
/* Launch on an external cudaStream_t (passed as void*); NULL = engine's own stream. */
int svg_engine_set_stream(svg_engine* e, void* stream);
/* Options (10): "tile_qubits" (0 = auto), "tile_fwd" (forward-only tile qubits, 0 auto, -1 off),
   "low_qubits" (3..5: contiguous low qubits every generated-kernel tile holds), "reg_bits"
   (0 auto, 3 or 4: 2^bits amplitudes per thread per buffer), "max_gates_per_pass" (0 = auto),
   "kernel" (0 auto, 1 shared-memory tiles, 2 register tiles), "jit" (circuit-specialised
   register-tile kernels compiled at run time with NVRTC: 0 off, 1 auto = shards of >= 10 qubits,
   2 always), "emulate_transport" (virtual engines: run the NCCL data path with device copies),
   "profile" (1 = per-phase CUDA-event times in svg_stats), "checked" (generated kernels poison every
   shared-memory element they read with NaN and bounds-check global tile indices: a read
   ordering bug shows up as NaN in the results; debugging and tests only). */
int svg_engine_set_option(svg_engine* e, const char* key, int64_t value);

/* The hot path: one full adjoint sweep.  sums_out[num_params] receives the
 * complex per-parameter sums (accumulated over repeated references in the
 * reference's order: gates descending, local parameters ascending);
 * deriv_out[num_derivs] (optional, may be NULL) the per-occurrence terms;
 * energy_out the complex <psi|H|psi>.  Synchronous: returns when the host
 * outputs are written. */
int svg_reverse_sweep(svg_engine* e, const svg_problem* p, svg_c128* sums_out,
                      svg_c128* deriv_out, svg_c128* energy_out, svg_stats* stats);

/* Forward pass + observable only: <psi|H|psi> (reference expectation(),
 * svgrad/observable.py:114-116). derivs are ignored. */
int svg_expectation(svg_engine* e, const svg_problem* p, svg_c128* energy_out, svg_stats* stats);

/* Host-only planner introspection (no CUDA calls): the gate application
 * order grouped into HBM passes.  order_out[G], pass_start_out[G+1],
 * qmask_out[G] (tile qubits of each pass); sms = SM count to plan for (0: 148). */
int svg_plan_inspect(const svg_problem* p, int tile_qubits, int sms, int32_t* order_out,
                     int32_t* pass_start_out, uint64_t* qmask_out, int32_t* npasses_out,
                     int32_t* tile_qubits_out);

/* Host-only sharded schedule (no CUDA calls) for `shards` shards: steps are
 * passes (step_swap_out[j] == 0; gates order_out[step_start[j]..step_start[j+1]),
 * tile qubits qmask_out[j] over physical local positions) or qubit swaps
 * (step_swap_out[j] == ((gbit << 8) | lpos) + 1).  Arrays sized for
 * num_gates + 2 * num_gates steps (an upper bound). */
int svg_plan_schedule(const svg_problem* p, int shards, int tile_qubits, int sms, int32_t* order_out,
                      int32_t* step_start_out, int32_t* step_swap_out, uint64_t* qmask_out, int32_t* nsteps_out,
                      int32_t* tile_qubits_out);

#ifdef __cplusplus
}
#endif
#endif /* SVGRAD_B200_H */
