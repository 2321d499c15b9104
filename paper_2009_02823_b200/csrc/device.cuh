// Device-side data structures shared by the pass kernels and the engine.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace svgb {

constexpr int kMaxQubits = 40;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

enum OpKind : uint32_t {
  OP_APPLY_PAULI = 0,  // buf <- a*buf + b'*Psign buf          (b' = b * i^{n_y})
  OP_APPLY_MAT1 = 1,   // 2x2 on one tile bit
  OP_APPLY_MAT2 = 2,   // 4x4 on two tile bits (sub-index bit k <-> t_k)
  OP_IP_PAULI = 3,     // acc[slot] += <lam| (ka + kb' Psign) P_c |phi>
  OP_IP_MAT1 = 4,
  OP_IP_MAT2 = 5,
};

// One tile-local operation.  Masks are expressed in tile-local bit positions
// (xl/zl/cl) or in global positions for the non-tile qubits (zo/co), whose
// values are constant over a tile.
struct DevOp {
  uint32_t kind;
  uint32_t buf;     // 0: psi/phi, 1: lambda (apply ops)
  uint32_t xl, zl, cl;
  uint32_t t0, t1;  // tile-local target positions (MAT ops)
  uint32_t slot;    // derivative slot inside the pass (IP ops)
  uint64_t zo, co;
  uint32_t coef;    // index into the coefficient array (double2)
  uint32_t pad[3];
};
static_assert(sizeof(DevOp) == 64, "DevOp layout");

// One observable Pauli string inside an observable pass.
struct DevTerm {
  double2 c;        // coeff * i^{n_y}
  uint32_t xl, zl;  // tile-local flip / sign masks
  uint64_t zo;      // sign mask on non-tile qubits
};
static_assert(sizeof(DevTerm) == 32, "DevTerm layout");

// Per-pass launch descriptor (passed by value).
struct PassDesc {
  int32_t n;             // qubits held by this device
  int32_t k;             // tile qubits
  int32_t b;             // contiguous low tile qubits (q[j] == j for j < b)
  int32_t op_begin, op_end;
  int32_t nslots;        // derivative slots (reverse) -- accumulators per CTA
  uint64_t rest;         // non-tile qubit mask (tile id bits are deposited here)
  int64_t part_off;      // this pass's slice of the partials buffer
  int32_t accumulate;    // observable pass: lambda += (1) or lambda = (0)
  int32_t untiled;       // observable pass over full-width masks (no tile)
  uint8_t q[kMaxQubits]; // tile qubits ascending
};

// Entry of the finalize map: deterministic sum of `count` partials at `off`.
struct SumSpec {
  int64_t off;
  int64_t count;
};

}  // namespace svgb
