// Device-side data structures shared by the pass kernels and the engine.
#pragma once
#ifdef __CUDACC_RTC__  // run-time compiled pass kernels (jit.cpp): no host headers
typedef unsigned char uint8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#else
#include <cstdint>
#include <cuda_runtime.h>
#endif

namespace svgb {

constexpr int kMaxQubits = 40;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRegBits = 3;  // amplitudes per thread per buffer = 2^kRegBits (register-tile passes)

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
  int32_t seg_begin, seg_end;  // register-tile passes: segment range
  int32_t smem_tiles;    // register-tile passes: 1 if the pass stages tiles in shared memory
  int32_t thread_acc;    // register-tile reverse passes: per-thread inner-product accumulators
  int32_t acc_shift;     // thread_acc: each accumulator combines 2^acc_shift adjacent lanes (butterfly)
  int32_t pad1;
  // Sharded state: this shard's rank bits in the physical amplitude index
  // (ORed into the tile base for Z-signs and controls, never for addressing),
  // and for observable passes the flip pattern on the rank bits of the source
  // shard (the partner whose amplitudes feed lambda).
  uint64_t rank_bits;
  uint64_t xglob;
  uint8_t q[kMaxQubits]; // tile qubits ascending
};

// ---- register-tile passes (kernels_reg.cu) ----
//
// A register-tile pass keeps each thread's share of the tile in registers:
// thread (warp w, lane l) holds 2^R amplitudes per buffer whose
// SEGMENT-LOCAL index is  t = l | j << 5 | w << (5 + R)  (j = register slot).
// Lane bits are always tile positions 0..4 (global qubits 0..4, so global
// loads/stores are 512-byte coalesced rows); each segment chooses which tile
// positions are register bits and which are warp bits.  Gates may flip lane
// bits (warp shuffles) and register bits (register permutations) but never
// warp bits; between segments the tile is transposed through shared memory.

// Every register op is a Pauli-form operator with real a and real-or-imaginary
// b' (all rotations, X/Y/Z, CX..., daggers of those):
//     new[t] = a v[t] + bb * (-1)^s(t) * (i^BI) v[t ^ x]
// where s(t) = parity((t ^ x) & z) ^ parity(base & zo).  The sign of the
// register part of t is precomputed per register slot (smask), so the device
// only adds the lane/warp part.  Controls likewise (cmask + clw).
enum RegOpKind : uint32_t {
  ROP_FWD = 0,  // psi <- op psi                                            (forward)
  ROP_REV = 1,  // [slot += <lam| K' |phi>]; phi <- op phi; lam <- op lam    (reverse: for a
                // unitary Pauli-form gate the rewind U^-1 and the adjoint U^dag coincide)
};
enum RegOpFlags : uint32_t {
  RF_IP1 = 1u,    // ROP_REV: accumulate one real component q = Re(conj(lam) sel(P phi))
  RF_IP3 = 2u,    // ROP_REV: accumulate the full complex z and z2 = <lam|phi> (complex / diag K')
  RF_BI = 4u,     // partner multiplied by i in the update (b' imaginary)
  RF_KBI = 8u,    // RF_IP1: select -i * partner (Im part) for the inner product
  RF_CTRL = 16u,  // op has controls inside the tile
};
enum RegOpShape : uint32_t {
  RS_DIAG = 0,   // no flip
  RS_LANE = 1,   // flip on lane bits only (warp shuffles)
  RS_REG = 2,    // flip on exactly one register bit (xr) -> register pairs
};

struct RegOp {
  uint32_t variant;   // flat code-path id (kernels_reg.cu run_variant)
  uint32_t flags, shape;
  uint32_t xl;        // lane flip mask
  uint32_t xr;        // register flip mask (one bit) for RS_REG
  uint32_t zlw;       // sign mask on lane | warp bits (segment-local)
  uint32_t clw;       // control mask on lane | warp bits (segment-local)
  uint32_t smask;     // bit j: parity((j ^ xr) & z_reg)     (register part of the partner sign)
  uint32_t cmask;     // bit j: (j & c_reg) == c_reg        (register part of the control test)
  uint32_t slot;
  uint64_t zo, co;    // non-tile (global) sign / control masks
  double a, bb;       // operator coefficients (see above)
  double kr;          // RF_IP1: contribution = kr * q (real part only)
  double2 ka, kb;     // RF_IP3: contribution = kb' z + ka z2
};
static_assert(sizeof(RegOp) == 112, "RegOp layout");

enum SegKind : int32_t { SEG_REG = 0, SEG_SMEM = 1 };

struct SegDesc {
  int32_t kind;
  int32_t op_begin, op_end;  // RegOps (SEG_REG) or DevOps (SEG_SMEM)
  int32_t same_map;          // SEG_REG: identical layout to the previous register segment
  uint8_t regpos[8];         // tile positions of register bits
  uint8_t warppos[8];        // tile positions of warp bits
  double scale;              // SEG_REG: deferred scale C of the register tile at the segment's end
                             // (product of the scaled ops' a since the last flush; kernels_reg.cu upd)
  uint8_t lanepos[8];        // tile positions of lane bits 0..4 (0,1,2,3,4 unless a free-lane plan)
};
static_assert(sizeof(SegDesc) == 48, "SegDesc layout");

// One pass of a product term's pipeline (k_prod_pass): the 2x2 factors whose
// qubits sit in this pass's tile, applied one after the other as butterflies
// over the shared-memory tile (Walsh-Hadamard for H).  Not last: the tile goes
// to the product buffer; last: lambda (+)= scalar * tile and the energy partial.
constexpr int kMaxProdFactors = 16;
struct ProdFactors {
  int32_t n;     // factors in this pass
  int32_t last;  // 1: accumulate into lambda (d.accumulate) with the energy partial
  uint32_t pos[kMaxProdFactors];            // tile-local positions
  double2 m[kMaxProdFactors][4];            // row-major 2x2 matrices
};

// Entry of the finalize map: deterministic sum of `count` partials at `off`.
struct SumSpec {
  int64_t off;
  int64_t count;
};

}  // namespace svgb
