// Circuit-specialised register-tile pass kernels, generated and compiled at
// run time (NVRTC, sm_100a).
//
// The interpreted kernel (kernels_reg.cu) reads each pass's program -- its
// segments (register layouts, transposes, shared-memory segments) and its
// register ops (variant id, masks, slot, coefficients) -- from memory and
// dispatches every op through a jump table, which costs decode instructions,
// register shuffling at the dispatch join, and instruction-cache misses.
// Here the same program is emitted as straight-line CUDA: the structure
// (variants, masks, layouts, slots) becomes template arguments and literals,
// only the theta-dependent numbers (operator coefficients, inner-product
// weights, deferred scales) stay runtime values -- kernel parameters, read
// from the constant bank.  Passes with identical structure (repeated circuit
// layers) share one kernel; kernels are cached per process.
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "device.cuh"

namespace svgb {

// One register-tile launch as the interpreter sees it.
struct JitPass {
  int R = 4, nb = 1, k = 0, nloc = 0, threads = 0;
  int nslots = 0;
  bool thread_acc = false, tiles = false;
  int acc_shift = 0;                 // thread_acc: lanes combined per accumulator (log2)
  bool scale_carry = false;          // deferred scale carried across layout changes (no shared-memory segments)
  bool checked = false;              // checked mode: shared-memory reads poison what they read, global indices
                                     // bounds-checked (reg_ops.cuh; debugging and tests only)
  int lowb = 5;                      // tile positions 0..lowb-1 are qubits 0..lowb-1 (contiguous global rows)
  uint64_t rest = 0;
  const uint8_t* q = nullptr;        // tile qubits (PassDesc.q)
  const uint8_t* swz = nullptr;      // shared-memory swizzle columns per tile position (engine.cu Swizzle)
  const SegDesc* segs = nullptr;     // the pass's segments
  int nsegs = 0;
  const RegOp* rops = nullptr;       // the pass's register ops (rops[0] is op_begin)
  int op_begin = 0;
};

// One tiled observable pass (k_obs_pass's work) for the generator.
struct JitObsPass {
  int k = 0, b = 0, nloc = 0, threads = 256;
  uint64_t rest = 0;
  const uint8_t* q = nullptr;
  const DevTerm* terms = nullptr;  // sorted by tile flip mask
  int nterms = 0;
  bool accumulate = false, remote = false;
};

// Where parameter c[i] comes from, relative to the pass.
struct CoefRef {
  enum Kind : uint8_t { A, BB, KR, KAX, KAY, KBX, KBY, SCALE, TRE, TIM, KRRUN } kind;
  int index;    // register op (relative to op_begin) or segment (relative to seg_begin)
  int aux = 0;  // KRRUN: first op of the fused diagonal run (kr rescaled to the run's start)
};

struct JitKernel {
  cudaKernel_t fn = nullptr;
  int regs = 0;
  size_t smem = 0;                 // dynamic shared memory per CTA
  std::vector<CoefRef> coefs;      // fill order of the parameter block's c[]
  std::vector<int> dop_segs;       // shared-memory segments whose DevOp base is a parameter
  uint64_t device_mask = 0;        // devices whose kernel attributes are set
  int blocks_per_sm = 0;           // occupancy (same for every B200), 0 = not queried yet
};

struct JitProgram {
  std::string src;
  std::vector<CoefRef> coefs;
  std::vector<int> dop_segs;
  size_t smem = 0;
};

// Parameter block prefix of every generated kernel (then int64 dop[], double c[]).
struct JitArgsHead {
  double2* b0;
  double2* b1;
  const DevOp* ops;
  const double2* coef;
  double2* partials;
  int64_t part_off;
  uint64_t rank_bits;
  uint64_t t0, t1;  // tile range of this launch: [0, 2^(nloc-k)) or one chunk of it
};

// Parameter block of a generated observable pass (then double c[]).
struct JitObsArgsHead {
  const double2* psi;
  const double2* src;
  double2* lam;
  double2* partials;
  int64_t part_off;
  uint64_t rank_bits;
  uint64_t xglob;
};

bool jit_available(std::string* why);
std::vector<std::shared_ptr<JitKernel>> jit_get_obs(const std::vector<JitObsPass>& passes, int device);
std::vector<unsigned char> jit_obs_args(const JitKernel& kern, const JitObsArgsHead& head, const DevTerm* terms);
JitProgram jit_generate(const JitPass& p);
// Kernels for the passes: cache hits by structural key; misses are generated
// and compiled (in parallel), then cached.  Throws std::runtime_error on compile / load failure.
// device < 0: dry run -- generate and compile every distinct structure, load nothing, return {}.
std::vector<std::shared_ptr<JitKernel>> jit_get(const std::vector<JitPass>& passes, int device);
// Parameter block for one launch.
std::vector<unsigned char> jit_args(const JitKernel& kern, const JitArgsHead& head, const SegDesc* segs,
                                    const RegOp* rops);
size_t jit_cache_size();

}  // namespace svgb
