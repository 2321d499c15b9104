// Engine + C-ABI entry points (include/svgrad_b200.h).
//
// One svg_reverse_sweep call == the reference's _reverse_sweep
// (svgrad/gradients.py:128-173):
//   1. plan      -- group gates into tile passes (plan.cpp), lower each gate
//                   and derivative generator to tile-local DevOps;
//   2. upload    -- one packed H2D copy of the op/coefficient/term tables;
//   3. init      -- psi = |basis> (memset + 1 store) or H2D of the host input;
//   4. forward   -- k_fwd_pass per forward pass              (:149-150)
//   5. observable-- k_obs_pass per term pass -> lambda, energy (:153-156)
//   6. reverse   -- k_rev_pass per pass, descending           (:158-168)
//   7. finalize  -- fixed-order partial sums, one D2H of (A+1) complex values;
//                   host accumulates sums[param_ref] in the reference order.
// The device state is exactly two complex128 buffers (psi/phi and lambda):
// the reference's probe clones (A+2 clones per call) do not exist here.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <deque>
#include <map>
#include <unordered_map>
#include <tuple>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/svgrad_b200.h"
#include "device.cuh"
#include "hash128.h"
#include "jit.h"
#include "kernels.h"
#include "nccl_shim.h"
#include "plan.h"

using namespace svgb;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

struct CudaError : std::runtime_error {
  cudaError_t code;
  CudaError(cudaError_t c, const char* what)
      : std::runtime_error(std::string(what) + ": " + cudaGetErrorString(c)), code(c) {}
};
// Generating / compiling / loading a circuit-specialised kernel failed (NVRTC
// missing or too old for sm_100a, load error): auto mode re-lowers for the
// interpreted kernels; forced mode (jit = 2) reports SVG_ECUDA.
struct JitFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct InvalidArg : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(call)                                  \
  do {                                            \
    cudaError_t _e = (call);                      \
    if (_e != cudaSuccess) throw CudaError(_e, #call); \
  } while (0)

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
inline double2 d2(const svg_c128& c) { return make_double2(c.re, c.im); }
inline double2 cm(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
// i^n
inline double2 ipow(int n) {
  switch (((n % 4) + 4) % 4) {
    case 0: return make_double2(1, 0);
    case 1: return make_double2(0, 1);
    case 2: return make_double2(-1, 0);
    default: return make_double2(0, -1);
  }
}

struct DeviceBuf {
  void* ptr = nullptr;
  size_t cap = 0;
  void reserve(size_t bytes) {
    if (bytes <= cap) return;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&ptr, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw CudaError(e, "cudaMalloc");
    }
    cap = bytes;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};
struct HostBuf {
  void* ptr = nullptr;
  size_t cap = 0;
  void reserve(size_t bytes) {
    if (bytes <= cap) return;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    cap = 0;
    CK(cudaMallocHost(&ptr, bytes));
    cap = bytes;
  }
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

enum LaunchKind { L_SMEM_FWD, L_SMEM_REV, L_OBS, L_OBS_DIRECT, L_REG, L_SWAP, L_FETCH, L_PROD };

// Shared-memory swizzle of a pass's transposes: element e of a tile lives at
// e ^ sum_{p >= 3, bit p of e set} col[p] (3-bit columns, bits 0..2).  A warp's
// 16-byte accesses are conflict-free when the columns of the tile positions on
// lane bits 0..2 are linearly independent (8 distinct 16-byte bank groups per
// quarter warp).  Positions 0..2 have columns 1, 2, 4 (identity), so the global
// layout (lanes on positions 0..4) is conflict-free for every choice.
struct Swizzle {
  uint8_t col[32] = {1, 2, 4};
};

struct Launch {
  PassDesc d;
  int grid = 0;
  size_t smem = 0;
  int kind = L_SMEM_FWD;
  int nb = 1;       // L_REG: buffers in the pass (1 forward, 2 reverse)
  int threads = kThreads;
  int R = 3;           // L_REG: register bits
  bool tiles = false;  // L_REG: stages the tile through shared memory
  int gbit = 0, lpos = 0;  // L_SWAP: rank bit <-> local position
  std::shared_ptr<JitKernel> jit;  // L_REG: circuit-specialised kernel (jit.cu), or null: interpreter
  Swizzle swz;                     // L_REG: shared-memory swizzle of the pass's transposes
  // L_PROD: this pass's factors; first pass reads psi (or the partner shard), later
  // ones the product buffer; the last one's scalar per source shard is
  // coeff * sum_j w_j (-1)^popcount(src rank bits & zg_j) (rank-bit factors in Pauli form)
  ProdFactors prod = {};
  bool prod_first = false;
  double2 prod_coeff = {0.0, 0.0};
  std::vector<std::pair<uint64_t, double2>> prod_z;
};

// Everything a sweep needs on the host side, built from one svg_problem.
struct Lowered {
  int n = 0, nloc = 0, k = 0, b = 0;
  int swaps = 0, obs_kernels = 0;
  int64_t swap_bytes = 0;  // bytes each shard exchanges (swaps both ways + partner fetches)
  bool reg = false;  // register-tile kernels in use
  bool free_lanes_used = false;  // some pass has a segment off the global lane layout (generated kernels only)
  bool fwd_early = false;        // forward launches handed to lower()'s fwd_ready callback (already launched)
  bool jit_planned = false;      // register passes planned for the generated kernels (deferred scale carried
                                 // across layout changes, see JitPass.scale_carry)
  int R = 3;         // their register bits
  std::vector<DevOp> ops;
  std::vector<double2> coef;
  std::vector<DevTerm> terms;
  std::vector<RegOp> rops;
  std::vector<SegDesc> segs;
  std::vector<SumSpec> sums;  // [num_derivs] derivative terms, then [1] energy
  std::vector<Launch> fwd, obs, rev;
  int64_t partial_count = 0;
  int64_t pass_bytes = 0;
};

// Derivative generator in both bases: `pre` acts on the state before the
// gate (the ABI's basis 0, the reference's probe order), `post` on the state
// after it (basis 1; what the register kernels fuse with the rewind).
struct Gen {
  svg_c128 pre[16];
  svg_c128 post[16];
};

}  // namespace

struct svg_engine {
  int device = 0;
  int sms = 148;
  size_t max_smem = 0;
  size_t max_smem_sm = 233472;  // shared memory per SM (B200: 228 KB)
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int64_t opt_tile = 0, opt_profile = 0, opt_max_items = 0, opt_kernel = 0, opt_reg_bits = 0;  // reg bits 0: auto
  int64_t opt_checked = 0;  // generated kernels in checked mode (reg_ops.cuh SVGB_CHECK / poison2)
  // virtual engines: run the NCCL-mode data path (half-shard pack -> copy ->
  // unpack, partner fetch into scratch) with device copies as the transport
  int64_t opt_emulate_transport = 0;
  // circuit-specialised register-tile kernels (jit.cu): 0 off, 1 auto (shards of
  // >= kJitMinQubits qubits), 2 always
  int64_t opt_jit = 1;
  int64_t opt_tile_fwd = 0;      // forward-only tile qubits (one shard, generated kernels): 0 auto (k+1), -1 off
  int64_t opt_slot_cap = 1;      // cap a pass's derivative slots at the per-thread accumulator budget
  int64_t opt_windows = 1;       // pass planner: also try windows of contiguous qubits (plan_best_pass)
  int64_t opt_low_qubits = 4;    // generated kernels: contiguous low qubits every tile holds (3..5)
  mutable std::string jit_error;
  int jit_dry_run = 0;             // svg_debug_jit_check (1), svg_debug_plan_stats (2: no compile)
  mutable double plan_stats[16] = {};
  mutable int jit_dry_count = 0;
  // occupancy queries are driver calls: memoised per (kernel kind, R, threads, smem)
  mutable std::map<std::tuple<int, int, int, size_t>, int> occ_memo;
  // segment plans are pure functions of a pass's flip / touch / dense pattern
  mutable std::unordered_map<Key128, std::vector<Segment>, Key128Hash> seg_memo;
  mutable std::unordered_map<Key128, std::pair<std::shared_ptr<const std::vector<Segment>>, Swizzle>, Key128Hash> choice_memo;
  mutable std::unordered_map<Key128, std::shared_ptr<const std::pair<std::vector<Step>, std::vector<int>>>, Key128Hash> plan_memo;  // why auto mode fell back to the interpreted kernels
  DeviceBuf psi, lam, partials, blob, results, scratch, gathered, prodbuf;
  HostBuf hblob, hres;
  // sharding: the state is split over 2^shard_bits shards by its top physical
  // qubits; this engine holds `shards_local` of them (virtual shards on one
  // device), or exactly one (rank `rank` of an NCCL communicator)
  int shard_bits = 0;
  int shards_local = 1;
  int rank = 0;
  NcclComm comm = nullptr;
  cudaEvent_t ev[6] = {};
  cudaEvent_t blob_ev = nullptr;  // the last table upload from the pinned staging buffer
  // chunked host input (one shard, >= kChunkMinQubits): copies on their own stream,
  // one event per chunk; the leading forward passes run chunk by chunk behind them
  static constexpr int kInputChunks = 16;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t chunk_ev[kInputChunks] = {};
  cudaEvent_t enter_ev = nullptr;
};

namespace {

void validate(const svg_problem* p) {
  if (!p) throw InvalidArg("null problem");
  const int n = p->num_qubits;
  if (n < 1 || n > SVG_MAX_QUBITS) throw InvalidArg("num_qubits out of range");
  if (p->num_gates < 0 || p->num_derivs < 0 || p->num_terms < 0 || p->num_params < 0 || p->num_product_terms < 0 ||
      p->num_factors < 0 || p->num_terms + p->num_product_terms < 1)
    throw InvalidArg("negative table size or empty observable");
  if ((p->num_gates && !p->gates) || (p->num_derivs && !p->derivs) || (p->num_terms && !p->terms) ||
      (p->num_product_terms && !p->product_terms) || (p->num_factors && !p->factors))
    throw InvalidArg("null table pointer");
  const uint64_t full = (n == 64) ? ~0ull : ((1ull << n) - 1);
  int d = 0;
  for (int i = 0; i < p->num_gates; ++i) {
    const svg_gate& g = p->gates[i];
    if (g.ntargets < 1 || g.ntargets > 2) throw InvalidArg("gate " + std::to_string(i) + ": 1 or 2 targets");
    uint64_t tm = 0;
    for (int j = 0; j < g.ntargets; ++j) {
      if (g.targets[j] < 0 || g.targets[j] >= n) throw InvalidArg("gate " + std::to_string(i) + ": target out of range");
      tm |= 1ull << g.targets[j];
    }
    if (__builtin_popcountll(tm) != g.ntargets) throw InvalidArg("gate " + std::to_string(i) + ": duplicate targets");
    if ((g.ctrl_mask & ~full) || (g.ctrl_mask & tm)) throw InvalidArg("gate " + std::to_string(i) + ": bad controls");
    if (g.form == SVG_FORM_PAULI) {
      if ((g.x_mask | g.z_mask) & ~tm) throw InvalidArg("gate " + std::to_string(i) + ": Pauli masks outside targets");
    } else if (g.form != SVG_FORM_MAT) {
      throw InvalidArg("gate " + std::to_string(i) + ": unknown form");
    }
    for (int j = 0; j < g.nderiv; ++j, ++d) {
      if (d >= p->num_derivs) throw InvalidArg("derivative table shorter than sum of arities");
      const svg_deriv& dv = p->derivs[d];
      if (dv.gate != i) throw InvalidArg("derivative table not gate-major");
      if (dv.param_ref < 0 || dv.param_ref >= p->num_params) throw InvalidArg("param_ref out of range");
      if (dv.form != g.form) throw InvalidArg("derivative form differs from its gate's form");
      if (dv.basis != 0 && dv.basis != 1) throw InvalidArg("derivative basis must be 0 or 1");
    }
  }
  if (d != p->num_derivs) throw InvalidArg("derivative table longer than sum of arities");
  for (int t = 0; t < p->num_terms; ++t) {
    const svg_pauli_term& tm = p->terms[t];
    if ((tm.x_mask | tm.z_mask) & ~full) throw InvalidArg("observable term outside register");
  }
  for (int t = 0; t < p->num_product_terms; ++t) {
    const svg_product_term& pt = p->product_terms[t];
    if (pt.first_factor < 0 || pt.num_factors < 0 || pt.first_factor + pt.num_factors > p->num_factors)
      throw InvalidArg("product term " + std::to_string(t) + ": factor range outside the factor table");
    uint64_t seen = 0;
    for (int f = pt.first_factor; f < pt.first_factor + pt.num_factors; ++f) {
      const int q = p->factors[f].qubit;
      if (q < 0 || q >= n || ((seen >> q) & 1))
        throw InvalidArg("product term " + std::to_string(t) + ": factor qubit out of range or repeated");
      seen |= 1ull << q;
    }
  }
  if (!p->input_amps && (p->input_basis < 0 || static_cast<uint64_t>(p->input_basis) > full))
    throw InvalidArg("basis index out of range");
}

struct TileMap {
  uint64_t qmask;
  int pos[SVG_MAX_QUBITS];
  uint32_t local(uint64_t m) const {
    uint32_t r = 0;
    for (uint64_t v = m & qmask; v; v &= v - 1) r |= 1u << pos[__builtin_ctzll(v)];
    return r;
  }
};

TileMap tile_map(uint64_t qmask) {
  TileMap tm;
  tm.qmask = qmask;
  int j = 0;
  for (int q = 0; q < SVG_MAX_QUBITS; ++q) tm.pos[q] = ((qmask >> q) & 1) ? j++ : -1;
  return tm;
}

PassDesc make_desc(int n, int k, uint64_t qmask) {
  PassDesc d;
  std::memset(&d, 0, sizeof(d));
  d.n = n;
  d.k = k;
  int j = 0;
  for (int q = 0; q < n; ++q)
    if ((qmask >> q) & 1) d.q[j++] = static_cast<uint8_t>(q);
  int b = 0;
  while (b < k && d.q[b] == b) ++b;
  d.b = b;
  const uint64_t full = (1ull << n) - 1;
  d.rest = full & ~qmask;
  return d;
}

// Emit one tile-local op for operator `c` (PAULI: a,b; MAT: matrix) of gate g.
void emit_op(Lowered& L, const TileMap& tm, const svg_gate& g, uint32_t kind_base, uint32_t buf,
             const svg_c128* c, uint32_t slot) {
  DevOp op;
  std::memset(&op, 0, sizeof(op));
  op.buf = buf;
  op.slot = slot;
  op.cl = tm.local(g.ctrl_mask);
  op.co = g.ctrl_mask & ~tm.qmask;
  op.coef = static_cast<uint32_t>(L.coef.size());
  if (g.form == SVG_FORM_PAULI) {
    op.kind = kind_base + 0;
    op.xl = tm.local(g.x_mask);
    op.zl = tm.local(g.z_mask);
    op.zo = g.z_mask & ~tm.qmask;
    L.coef.push_back(d2(c[0]));
    L.coef.push_back(cm(d2(c[1]), ipow(g.n_y)));  // coefficient of the sign-only permutation
  } else if (g.ntargets == 1) {
    op.kind = kind_base + 1;
    op.t0 = static_cast<uint32_t>(tm.pos[g.targets[0]]);
    for (int i = 0; i < 4; ++i) L.coef.push_back(d2(c[i]));
  } else {
    op.kind = kind_base + 2;
    op.t0 = static_cast<uint32_t>(tm.pos[g.targets[0]]);
    op.t1 = static_cast<uint32_t>(tm.pos[g.targets[1]]);
    for (int i = 0; i < 16; ++i) L.coef.push_back(d2(c[i]));
  }
  L.ops.push_back(op);
}

// (c0 I + c1 P)(d0 I + d1 P) with P^2 = I
void pauli_mul(const svg_c128* x, const svg_c128* y, svg_c128* out) {
  const double2 x0 = d2(x[0]), x1 = d2(x[1]), y0 = d2(y[0]), y1 = d2(y[1]);
  const double2 a = cm(x0, y0), b = cm(x1, y1), c = cm(x0, y1), d = cm(x1, y0);
  out[0] = svg_c128{a.x + b.x, a.y + b.y};
  out[1] = svg_c128{c.x + d.x, c.y + d.y};
  for (int i = 2; i < 16; ++i) out[i] = svg_c128{0.0, 0.0};
}

void mat_mul(const svg_c128* x, const svg_c128* y, int dim, svg_c128* out) {
  svg_c128 r[16] = {};
  for (int i = 0; i < dim; ++i)
    for (int j = 0; j < dim; ++j) {
      double2 acc = make_double2(0.0, 0.0);
      for (int k = 0; k < dim; ++k) {
        const double2 t = cm(d2(x[i * dim + k]), d2(y[k * dim + j]));
        acc.x += t.x;
        acc.y += t.y;
      }
      r[i * dim + j] = svg_c128{acc.x, acc.y};
    }
  for (int i = 0; i < 16; ++i) out[i] = r[i];
}

Gen make_gen(const svg_gate& g, const svg_deriv& dv) {
  Gen gen;
  const bool post = dv.basis == 1;
  const svg_c128* given = dv.k;
  svg_c128* other = post ? gen.pre : gen.post;
  std::memcpy(post ? gen.post : gen.pre, given, sizeof(gen.pre));
  // pre = post * U ; post = pre * R   (R = U^-1 on the control subspace)
  const svg_c128* right = post ? g.fwd : g.rewind;
  if (g.form == SVG_FORM_PAULI)
    pauli_mul(given, right, other);
  else
    mat_mul(given, right, 1 << g.ntargets, other);
  return gen;
}

// Segment-local bit of each tile position for a register segment.
struct SegLocal {
  int R = 3;  // register bits of the segment layout
  uint8_t bit[32];
  uint32_t conv(uint32_t tile_mask) const {
    uint32_t r = 0;
    for (uint32_t v = tile_mask; v; v &= v - 1) r |= 1u << bit[__builtin_ctz(v)];
    return r;
  }
};

static bool independent3(uint32_t a, uint32_t b, uint32_t c) {
  return a && b && c && a != b && c != a && c != b && c != (a ^ b);
}

// Lane order for a lane set: three positions with independent columns first
// (lane bits 0..2), preferring low positions; false if there are none.
static bool order_lanes(uint32_t laneset, const Swizzle& sw, uint8_t out[5]) {
  int pos[5], np = 0;
  for (uint32_t v = laneset; v && np < 5; v &= v - 1) pos[np++] = __builtin_ctz(v);
  for (int a = 0; a < np; ++a)
    for (int b = a + 1; b < np; ++b)
      for (int c = b + 1; c < np; ++c)
        if (independent3(sw.col[pos[a]], sw.col[pos[b]], sw.col[pos[c]])) {
          out[0] = uint8_t(pos[a]);
          out[1] = uint8_t(pos[b]);
          out[2] = uint8_t(pos[c]);
          int o = 3;
          for (int d = 0; d < np; ++d)
            if (d != a && d != b && d != c) out[o++] = uint8_t(pos[d]);
          return true;
        }
  for (int d = 0; d < np; ++d) out[d] = uint8_t(pos[d]);
  return false;
}

// Swizzle for a pass whose segments use these lane sets (identity when every
// segment keeps the global lanes).  Deterministic search; on failure the
// cyclic assignment (some 2-way bank conflicts).
static Swizzle choose_swizzle(const std::vector<uint32_t>& lanesets, int k) {
  Swizzle sw;
  bool all_std = true;
  for (uint32_t l : lanesets) all_std = all_std && l == 31u;
  if (all_std) return sw;
  uint32_t rng = 0x9e3779b9u;
  for (int t = 0; t < 256; ++t) {
    Swizzle c;
    for (int p = 3; p < k; ++p) {
      if (t == 0) {
        c.col[p] = uint8_t(((p - 3) % 7) + 1);
      } else {
        rng = rng * 1664525u + 1013904223u;
        c.col[p] = uint8_t(1 + (rng >> 24) % 7);
      }
    }
    bool ok = true;
    uint8_t tmp[5];
    for (uint32_t l : lanesets) ok = ok && order_lanes(l, c, tmp);
    if (ok) return c;
    if (t == 0) sw = c;
  }
  return sw;
}

SegDesc make_seg(int kind, uint32_t regmask, uint32_t lanemask, const Swizzle& swz, int k, int R, SegLocal* sl) {
  sl->R = R;
  SegDesc sd;
  std::memset(&sd, 0, sizeof(sd));
  sd.scale = 1.0;
  sd.kind = kind;
  uint8_t lp[5] = {0, 1, 2, 3, 4};
  if (lanemask != 31u) order_lanes(lanemask, swz, lp);
  for (int i = 0; i < 5; ++i) {
    sd.lanepos[i] = lp[i];
    sl->bit[lp[i]] = static_cast<uint8_t>(i);
  }
  int r = 0, w = 0;
  for (int pos = 0; pos < k; ++pos) {
    if ((lanemask >> pos) & 1) continue;
    if ((regmask >> pos) & 1) {
      sd.regpos[r] = static_cast<uint8_t>(pos);
      sl->bit[pos] = static_cast<uint8_t>(5 + r++);
    } else {
      sd.warppos[w] = static_cast<uint8_t>(pos);
      sl->bit[pos] = static_cast<uint8_t>(5 + R + w++);
    }
  }
  return sd;
}

// Smallest |a| whose 1/a the scaled register form may carry (|t| = |b/a| <= 1e3:
// the scaled form v + t P v has the same rounding error as a v + b P v, and the
// host keeps the deferred scale C of a tile inside [1e-60, 1]).
constexpr double kMinDeferredA = 1e-3;
constexpr double kMinDeferredC = 1e-60;
// Auto mode compiles circuit-specialised kernels for shards of at least this
// many qubits (measured 1.8-2x the interpreter's gradients/s from 10 qubits on;
// below 10 the first call's compile outweighs the few microseconds of work).
constexpr int kJitMinQubits = 10;
// Gates per register-tile pass.  With the window planner a pass holds a
// parallelogram of the circuit several layers deep, so the cap (with the slot
// cap below) sets the number of HBM passes: measured cfg 4 (n = 30) 0.94 / 1.01 /
// 1.05 / 1.06 gradients/s at 44 / 48 / 64 / 72 (36 / 30 / 27 / 25 passes per sweep),
// cfg 3 9.3 / 9.8 / 9.8 at 40 / 48 / 56 (its passes reach the slot cap first).
constexpr int kRegPassGates = 64;
// Forward passes (psi only, no accumulators, a third of the arithmetic per gate) on
// their own schedule: measured cfg 4 forward 226 / 204 / 207 / 209 ms at 64 / 80 / 96 / 128.
constexpr int kFwdPassGates = 80;
// States this large (per shard) stream HBM: generated kernels use 12-qubit tiles
// (a narrower reverse tile gets a forward schedule over k+1-qubit tiles).
constexpr int kWideTileQubits = 24;
// Host input states of at least this many qubits (one shard) are copied in chunks with
// the leading forward passes pipelined behind the copy (SVGB_CHUNK_MIN_QUBITS overrides: tests).
inline int chunk_min_qubits() {
  if (const char* v = std::getenv("SVGB_CHUNK_MIN_QUBITS")) return std::max(16, std::atoi(v));
  return 26;
}
// Segment-plan cost model in register-op units (a register rotation = 1): a lane
// flip is a warp shuffle of both buffers (forward: one), a layout change a
// shared-memory transpose.  Measured with tools/pass_model.py (round 1).
constexpr double kLaneCost = 3.7, kXposeCost = 5.3;        // reverse passes (phi and lambda)
constexpr double kFwdLaneCost = 5.0, kFwdXposeCost = 8.0;  // forward passes (psi only)

// One register op for gate g: operator coefficients `c` (a, b of a I + b P),
// optionally fused with the post-gate generator `kpost` into `slot`.
// `cs` is the register tile's deferred scale C (tile = state / C) before the op:
// an uncontrolled rotation runs in the scaled form  v + (b/a) P v  and multiplies
// C by a; its inner-product coefficients carry C^2 (phi and lambda share C).
void emit_rop(Lowered& L, const TileMap& tm, const SegLocal& sl, const svg_gate& g, uint32_t kind,
              const svg_c128* c, const svg_c128* kpost, uint32_t slot, bool real_sums, double* cs) {
  RegOp op;
  std::memset(&op, 0, sizeof(op));
  const int R = sl.R;
  const uint32_t regbits = ((1u << R) - 1u) << 5;
  const uint32_t xloc = sl.conv(tm.local(g.x_mask));
  const uint32_t zloc = sl.conv(tm.local(g.z_mask));
  const uint32_t cloc = sl.conv(tm.local(g.ctrl_mask));
  op.xl = xloc & 31u;
  op.xr = (xloc & regbits) >> 5;
  op.shape = xloc == 0 ? RS_DIAG : (op.xr == 0 ? RS_LANE : RS_REG);
  op.zlw = zloc & ~regbits;
  op.clw = cloc & ~regbits;
  const uint32_t zr = (zloc & regbits) >> 5, cr = (cloc & regbits) >> 5;
  for (uint32_t j = 0; j < (1u << R); ++j) {
    op.smask |= static_cast<uint32_t>(__builtin_popcount((j ^ op.xr) & zr) & 1) << j;
    op.cmask |= static_cast<uint32_t>((j & cr) == cr) << j;
  }
  if (cloc) op.flags |= RF_CTRL;
  op.zo = g.z_mask & ~tm.qmask;
  op.co = g.ctrl_mask & ~tm.qmask;
  const double2 ph = ipow(g.n_y);
  const double2 b = cm(d2(c[1]), ph);
  op.a = c[0].re;
  // BI: b' imaginary.  With b' == 0 either form works; pick the generator's
  // so the fused inner product can use the same compile-time variant.
  bool bi = b.x == 0.0 && b.y != 0.0;
  double2 kb = make_double2(0.0, 0.0), ka = kb;
  if (kpost) {
    ka = d2(kpost[0]);
    kb = cm(d2(kpost[1]), ph);
    if (b.x == 0.0 && b.y == 0.0) bi = kb.x == 0.0 && kb.y != 0.0;
  }
  if (bi) op.flags |= RF_BI;
  op.bb = bi ? b.y : b.x;
  if (kpost) {
    op.slot = slot;
    op.ka = ka;
    op.kb = kb;
    const bool diag = ka.x != 0.0 || ka.y != 0.0;
    // single-component inner product when only Re(sums) is needed and kb' is
    // real (Re(kb' z) = kb'.x Re z) or imaginary (Re(i k z) = -k Im z) --
    // the latter must coincide with the update's BI variant.
    if (real_sums && !diag && kb.y == 0.0 && !bi) {
      op.flags |= RF_IP1;
      op.kr = kb.x;
    } else if (real_sums && !diag && kb.x == 0.0 && bi) {
      op.flags |= RF_IP1 | RF_KBI;
      op.kr = -kb.y;
    } else {
      op.flags |= RF_IP3;
    }
  }
  // flat code-path id, see Pat<R> and run_variant in kernels_reg.cu
  const uint32_t P_DIAG = 0, P_DIAGZ = 1, P_LANE = 1 + R, P_REG = 2 + R, P_REGY = 2 + 2 * R, P_GDIAG = 2 + 3 * R,
                 P_GLANE = 3 + 3 * R, P_GREG = 4 + 3 * R, NP = 4 + 4 * R;
  uint32_t pattern;
  if (op.shape == RS_DIAG)
    pattern = zr == 0 ? P_DIAG : (__builtin_popcount(zr) == 1 ? P_DIAGZ + __builtin_ctz(zr) : P_GDIAG);
  else if (op.shape == RS_LANE)
    pattern = zr == 0 ? P_LANE : P_GLANE;
  else {
    const uint32_t b = __builtin_ctz(op.xr);
    pattern = zr == 0 ? P_REG + b : (zr == op.xr ? P_REGY + b : P_GREG + b);
  }
  // pure Pauli (X/Y/Z, CX, ...): a signed permutation without arithmetic
  const bool perm = op.a == 0.0 && std::fabs(op.bb) == 1.0 && !kpost;
  uint32_t mode = perm ? 2 + (bi ? 1 : 0) : (bi ? 1 : 0);  // forward kernel modes
  if (kind == ROP_REV) {                                    // reverse kernel modes
    if (op.flags & RF_IP3)
      mode = 2;
    else if (op.flags & RF_IP1)
      mode = bi ? 1 : 0;
    else if (perm)
      mode = 3 + (bi ? 1 : 0);
    else
      throw std::logic_error("parameter-free non-permutation Pauli op reached the register path");
  }
  // inner products see the tile before this op: scale by C^2
  const double c2 = (*cs) * (*cs);
  op.kr *= c2;
  op.ka = make_double2(op.ka.x * c2, op.ka.y * c2);
  op.kb = make_double2(op.kb.x * c2, op.kb.y * c2);
  bool ctrl = cloc != 0;
  if (!perm && !ctrl) {
    if (op.co == 0 && std::fabs(op.a) >= kMinDeferredA && std::fabs(*cs * op.a) >= kMinDeferredC) {
      // scaled form: v + t P v, C *= a
      op.bb /= op.a;
      *cs *= op.a;
    } else {  // controlled by a non-tile qubit (skipped on some tiles) or tiny a: unscaled form
      ctrl = true;
      op.flags |= RF_CTRL;
      op.cmask = (R >= 5) ? ~0u : ((1u << (1u << R)) - 1u);
      op.clw = 0;
    }
  }
  op.variant = pattern + NP * ((ctrl ? 1 : 0) + 2 * mode);
  L.rops.push_back(op);
}

// Whether a gate runs as a register op: Pauli form with a real a and a real or
// imaginary b' in all three operators, at most one parameter, and a flip that
// touches lanes only or exactly one non-lane tile position.
bool reg_capable(const svg_gate& g, uint32_t flip_tile) {
  if (g.form != SVG_FORM_PAULI || g.nderiv > 1) return false;
  for (int i = 0; i < 2; ++i)  // one reverse op serves phi and lambda: rewind must equal adjoint
    if (g.rewind[i].re != g.adjoint[i].re || g.rewind[i].im != g.adjoint[i].im) return false;
  const double2 ph = ipow(g.n_y);
  for (const svg_c128* c : {g.fwd, g.rewind, g.adjoint}) {
    const double2 b = cm(d2(c[1]), ph);
    if (c[0].im != 0.0 || (b.x != 0.0 && b.y != 0.0)) return false;
    // parameter-free ops must be signed permutations (the reverse kernel has no plain-rewind mode)
    if (g.nderiv == 0 && (c[0].re != 0.0 || std::fabs(b.x + b.y) != 1.0)) return false;
  }
  const uint32_t hi = flip_tile & ~31u;
  if (hi == 0) return true;
  return __builtin_popcount(hi) == 1 && (flip_tile & 31u) == 0;
}

std::vector<Segment> memo_segments(const svg_engine* e, const std::vector<uint32_t>& flips,
                                   const std::vector<uint32_t>& touch, const std::vector<char>& dense, int k,
                                   int regbits, bool free = false, int lowb = 5) {
  Hasher h;
  const int32_t head[] = {k, regbits, free ? 1 + lowb : 0, static_cast<int32_t>(flips.size())};
  h.pod(head);
  h.bytes(flips.data(), flips.size() * 4);
  h.bytes(touch.data(), touch.size() * 4);
  h.bytes(dense.data(), dense.size());
  const Key128 key = h.key();
  auto it = e->seg_memo.find(key);
  if (it != e->seg_memo.end()) return it->second;
  std::vector<Segment> segs =
      free ? plan_segments_free(flips, touch, k, regbits, lowb) : plan_segments(flips, touch, dense, k, regbits);
  if (e->seg_memo.size() > 16384) e->seg_memo.clear();
  e->seg_memo.emplace(key, segs);
  return segs;
}

// The gates of one pass step (pointers into the problem or into remapped copies).
struct GateList {
  std::vector<const svg_gate*> ptr;
  const svg_gate& operator[](size_t i) const { return *ptr[i]; }
  size_t size() const { return ptr.size(); }
  struct It {
    const svg_gate* const* p;
    const svg_gate& operator*() const { return **p; }
    It& operator++() {
      ++p;
      return *this;
    }
    bool operator!=(const It& o) const { return p != o.p; }
  };
  It begin() const { return It{ptr.data()}; }
  It end() const { return It{ptr.data() + ptr.size()}; }
};

// Physical copy of a gate under the logical -> physical qubit map of its step.
svg_gate physical_gate(const svg_gate& g, const std::vector<int>& l2p) {
  svg_gate q = g;
  for (int j = 0; j < g.ntargets; ++j) q.targets[j] = l2p[g.targets[j]];
  q.ctrl_mask = remap_mask(g.ctrl_mask, l2p);
  q.x_mask = remap_mask(g.x_mask, l2p);
  q.z_mask = remap_mask(g.z_mask, l2p);
  return q;
}

// Host-side phase timing of lower() (svg_debug_lower_timing).
thread_local double g_phase_ms[9];
thread_local std::chrono::steady_clock::time_point g_phase_t;
#define SVGB_PHASE(i)                                                                                  \
  do {                                                                                                 \
    const auto now_ = std::chrono::steady_clock::now();                                              \
    g_phase_ms[(i)-1] += std::chrono::duration<double, std::milli>(now_ - g_phase_t).count();        \
    g_phase_t = now_;                                                                                  \
  } while (0)

// fwd_ready (optional): called once the forward launches are complete and sized
// -- generated kernels only, no shared-memory segments -- so the caller can start
// them while the rest (observable, reverse sweep) is still being lowered.
Lowered lower(const svg_engine* e, const svg_problem* p, bool with_reverse,
              const std::function<void(Lowered&)>& fwd_ready = {}, bool interp_only = false) {
  g_phase_t = std::chrono::steady_clock::now();
  Lowered L;
  const int n = p->num_qubits;
  const int g = e->shard_bits;  // log2(shards): top g physical qubits select the shard
  const int nloc = n - g;
  if (nloc < 1) throw InvalidArg("more shards than amplitudes");
  const bool real_sums = (p->flags & SVG_FLAG_REAL_SUMS) != 0;
  L.n = n;
  L.nloc = nloc;
  // generated kernels (shards of >= kJitMinQubits): two tiles per SM suffice
  // (one CTA pair); wider tiles mean fewer passes (measured cfg 2: k 11 / R 4 6 % faster)
  const bool jit_expected = e->opt_jit == 2 || (e->opt_jit == 1 && nloc >= kJitMinQubits);
  L.k = choose_tile_qubits(nloc, static_cast<int>(e->opt_tile), e->sms, jit_expected ? 2 : 4);
  // HBM-resident states with generated kernels: 12-qubit tiles (one 256-thread CTA
  // per SM; fewer passes -- measured cfg 3 reverse -7 %, cfg 4 -9 %)
  if (e->opt_tile == 0 && jit_expected && nloc >= kWideTileQubits && (int64_t(1) << (nloc - 12)) >= 2ll * e->sms)
    L.k = 12;
  // small states (L2-resident, latency-bound passes): fewer, wider passes beat
  // tile balance -- measured cfg 2 structure, n = 12 / 14 / 16 / 18: best k =
  // 10 / 10 / 11 / 12 (2427 / 2134 / 1800 / 1490 gradients/s)
  if (e->opt_tile == 0 && jit_expected && nloc <= 18 && nloc > 10) L.k = std::max(10, std::min(12, nloc - 5));
  L.b = (nloc <= L.k) ? nloc : std::min(5, L.k - 2);
  if (g > 0 && L.b < 5 && nloc > L.k) throw InvalidArg("sharded engines need >= 7 qubits per shard");
  // register bits (amplitudes per thread per buffer = 2^R): auto = 4 for the
  // generated kernels (fewer ops per amplitude; measured cfg 2 / cfg 3) unless the
  // whole state is one tile -- then a pass is one CTA on one SM, and twice the warps
  // hide more latency (cfg 1: 6416 vs 5088 gradients/s at R = 3 / 4); the
  // interpreter keeps 3 for shards of <= 23 qubits (more threads per tile: better
  // latency hiding when a pass is only a few tile rounds)
  const int Rauto = (nloc <= 23 && !jit_expected) || (jit_expected && nloc <= L.k) ? 3 : 4;
  const int RB = e->opt_reg_bits ? static_cast<int>(e->opt_reg_bits) : Rauto;          // reverse passes
  const int RF = RB;  // forward passes
  L.R = RB;
  // thread count of a register-tile CTA: the interpreter's launch bounds, or 512
  // for the generated kernels (their launch bounds follow the thread count)
  auto fits = [&](int R) {
    return L.k - 5 - R >= 0 && (32 << (L.k - 5 - R)) <= (jit_expected ? 512 : reg_max_threads(R));
  };
  L.reg = e->opt_kernel != 1 && L.b >= 5 && fits(RB) && fits(RF);
  if (e->opt_kernel == 2 && !L.reg) throw InvalidArg("register-tile kernels need 5 + reg_bits .. 13 tile qubits");
  // free-lane plans and carried scales need the generated kernels (the
  // interpreter keeps lanes on tile positions 0..4)
  const bool jit_planned = L.reg && !interp_only && (e->opt_jit == 2 || (e->opt_jit == 1 && nloc >= kJitMinQubits)) &&
                           (e->jit_dry_run || jit_available(nullptr));
  L.jit_planned = jit_planned;
  // Generated kernels address the global tile through the lanes' physical qubits, so
  // their tiles need only qubits 0..low_qubits-1 (256-byte rows at 4) instead of
  // 0..4: more tile qubits free for the circuit.  cfg 4: 61 / 56 / 52 passes per
  // sweep at 5 / 4 / 3 low qubits, measured 0.708 / 0.758 / 0.714 gradients/s (at 3
  // the 128-byte rows cost more per pass than the 4 saved passes)
  if (jit_planned && nloc > L.k && e->opt_low_qubits < L.b) L.b = static_cast<int>(e->opt_low_qubits);
  PlanParams pp;
  pp.n = nloc;
  pp.k = L.k;
  pp.b = L.b;
  if (e->opt_max_items > 0)
    pp.max_items = static_cast<int>(e->opt_max_items);
  else if (L.reg)
    pp.max_items = kRegPassGates;
  pp.windows = e->opt_windows != 0;
  // Generated reverse kernels keep one inner-product accumulator per (slot, thread)
  // in shared memory next to the transpose tiles; past that budget lanes are
  // combined per op (a butterfly step each, measured 8 % per halving): cap the
  // parametrised gates of a pass at what fits (46 at k = 12 / 11 with R = 4).
  if (jit_planned && L.reg && e->opt_slot_cap) {
    const int threads = 32 << (L.k - 5 - RB);
    const int blocks = std::max(1, std::min(2, 256 / threads));
    const size_t share = std::min<size_t>(e->max_smem, size_t(e->max_smem_sm) / blocks - 1024);
    const size_t tiles_b = (sizeof(double2) << L.k) * 2;
    const size_t per_slot = size_t(threads) * sizeof(double) + sizeof(double2) * (threads / 32);
    if (share > tiles_b + 8 * per_slot) pp.max_derivs = std::min<int>(pp.max_derivs, int((share - tiles_b) / per_slot));
  }
  const int64_t S = int64_t(16) << nloc;  // bytes of one state shard

  std::vector<GateShape> logical(p->num_gates);
  for (int i = 0; i < p->num_gates; ++i) logical[i] = gate_shape(p->gates[i]);
  std::vector<int> l2p_final;
  // the schedule is a pure function of the gate shapes and plan parameters: memoised
  auto schedule = [&](const PlanParams& pq, std::vector<int>* l2p_out) {
    Hasher h;
    const int32_t head[] = {n, g, pq.n, pq.k, pq.b, pq.max_items, pq.max_derivs, pq.windows, static_cast<int32_t>(logical.size())};
    h.pod(head);
    for (const GateShape& sh : logical) {
      h.word(sh.flip);
      h.word(sh.touch);
      h.word(static_cast<uint64_t>(sh.nderiv));
    }
    const Key128 key = h.key();
    auto it = e->plan_memo.find(key);
    if (it != e->plan_memo.end()) {
      if (l2p_out) *l2p_out = it->second->second;
      return it->second;
    }
    std::vector<int> l2p;
    std::vector<Step> st = plan_schedule(logical, n, g, pq, &l2p);
    auto entry = std::make_shared<const std::pair<std::vector<Step>, std::vector<int>>>(std::move(st), std::move(l2p));
    if (e->plan_memo.size() > 64) e->plan_memo.clear();
    e->plan_memo.emplace(key, entry);
    if (l2p_out) *l2p_out = entry->second;
    return std::shared_ptr<const std::pair<std::vector<Step>, std::vector<int>>>(entry);
  };
  const auto sched = schedule(pp, &l2p_final);
  const std::vector<Step>& steps = sched->first;
  // The forward sweep only has to deliver psi at its end, so (one shard, generated
  // kernels) it runs its own schedule over larger tiles -- one buffer per tile
  // leaves room for 2^(k+1) amplitudes per CTA: fewer HBM passes.
  int kf = L.k;
  std::shared_ptr<const std::pair<std::vector<Step>, std::vector<int>>> sched_f;
  // (wider tiles, auto: states of >= kWideTileQubits qubits, whose passes stream HBM,
  // when the reverse tile is narrower than 12; smaller, L2-resident states are better
  // served by more, smaller tiles -- measured cfg 2).  The forward passes also carry no
  // inner-product accumulators, so the slot cap does not apply to them.
  if (g == 0 && jit_planned && nloc > L.k) {
    if (e->opt_tile_fwd > 0 || (e->opt_tile_fwd == 0 && nloc >= kWideTileQubits && L.k <= 11)) {
      kf = e->opt_tile_fwd > 0 ? static_cast<int>(e->opt_tile_fwd) : L.k + 1;
      kf = std::max(L.k, std::min({kf, nloc, 13}));
    }
    PlanParams pq = pp;
    pq.k = kf;
    pq.max_derivs = 1 << 20;
    if (e->opt_max_items <= 0) pq.max_items = kFwdPassGates;
    if (nloc >= kWideTileQubits || kf > L.k) sched_f = schedule(pq, nullptr);
  }
  const std::vector<Step>& fsteps = sched_f ? sched_f->first : steps;
  // physical gates per pass step, parallel to the step's items
  std::vector<GateList> pgates(steps.size());
  std::deque<svg_gate> pstore;  // remapped copies (only when the qubit map is not the identity)
  std::vector<std::vector<GateShape>> pshapes(steps.size());
  for (size_t si = 0; si < steps.size(); ++si) {
    if (steps[si].swap) continue;
    for (int gi : steps[si].pass.items) {
      bool ident = true;
      for (size_t q = 0; q < steps[si].l2p.size() && ident; ++q) ident = steps[si].l2p[q] == static_cast<int>(q);
      if (ident) {
        pgates[si].ptr.push_back(&p->gates[gi]);
      } else {
        pstore.push_back(physical_gate(p->gates[gi], steps[si].l2p));
        pgates[si].ptr.push_back(&pstore.back());
      }
      pshapes[si].push_back(gate_shape(pgates[si][pgates[si].size() - 1]));
    }
  }

  std::vector<GateList> pgates_fs;
  std::vector<std::vector<GateShape>> pshapes_fs;
  if (&fsteps != &steps) {  // one shard: identity qubit map
    pgates_fs.resize(fsteps.size());
    pshapes_fs.resize(fsteps.size());
    for (size_t si = 0; si < fsteps.size(); ++si)
      for (int gi : fsteps[si].pass.items) {
        pgates_fs[si].ptr.push_back(&p->gates[gi]);
        pshapes_fs[si].push_back(logical[gi]);
      }
  }
  const std::vector<GateList>& fpgates = &fsteps != &steps ? pgates_fs : pgates;
  const std::vector<std::vector<GateShape>>& fpshapes = &fsteps != &steps ? pshapes_fs : pshapes;

  std::vector<int> first_deriv(p->num_gates + 1, 0);
  for (int i = 0; i < p->num_gates; ++i) first_deriv[i + 1] = first_deriv[i] + p->gates[i].nderiv;
  SVGB_PHASE(1);
  std::vector<Gen> gens(p->num_derivs);
  for (int d = 0; d < p->num_derivs; ++d) gens[d] = make_gen(p->gates[p->derivs[d].gate], p->derivs[d]);

  SVGB_PHASE(2);
  // segments per pass (register path)
  using SegsPtr = std::shared_ptr<const std::vector<Segment>>;
  std::vector<SegsPtr> psegs(steps.size()), psegs_f(fsteps.size());
  std::vector<Swizzle> pswz(steps.size()), pswz_f(fsteps.size());
  // free-lane plans also need tile staging (a first segment off the global
  // layout reads its tile from the staged copy)
  const bool free_lanes = jit_planned;
  // Tile rows are 2^L.b contiguous amplitudes: a layout whose lanes include tile
  // positions 0..lowb-1 loads and stores whole rows whatever its other lanes hold,
  // so (generated kernels, L.b < 5) it needs no transpose back to positions 0..4
  const int lowb = std::min(5, L.b);
  const uint32_t lowmask = (1u << lowb) - 1u;
  // segments of one pass at tile width kk with R register bits: the fixed-lane
  // plan, or the free-lane plan when the cost model prefers it (lc: lane op,
  // xc: layout change, in register-op units)
  auto pass_segments = [&](const Pass& ps, const GateList& gl, const std::vector<GateShape>& shp, int kk, int R,
                           double lc, double xc, SegsPtr* outp, Swizzle* swz) {
    const TileMap tm = tile_map(ps.qmask);
    std::vector<uint32_t> flips(ps.items.size()), touch(ps.items.size());
    std::vector<char> dense(ps.items.size());
    for (size_t j = 0; j < ps.items.size(); ++j) {
      flips[j] = tm.local(shp[j].flip);
      touch[j] = tm.local(shp[j].touch);
      dense[j] = !reg_capable(gl[j], flips[j]);
    }
    // the choice (plan + swizzle) is memoised per pass structure and cost model
    Hasher h;
    const int32_t head[] = {kk, R, free_lanes ? 1 + lowb : 0, static_cast<int32_t>(flips.size())};
    h.pod(head);
    h.pod(lc);
    h.pod(xc);
    h.bytes(flips.data(), flips.size() * 4);
    h.bytes(touch.data(), touch.size() * 4);
    h.bytes(dense.data(), dense.size());
    const Key128 ck = h.key();
    auto hit = e->choice_memo.find(ck);
    if (hit != e->choice_memo.end()) {
      *outp = hit->second.first;
      *swz = hit->second.second;
      for (const Segment& sg : **outp) L.free_lanes_used = L.free_lanes_used || sg.lanemask != 31u;
      return;
    }
    auto chosen = std::make_shared<std::vector<Segment>>(memo_segments(e, flips, touch, dense, kk, R));
    std::vector<Segment>* out = chosen.get();
    bool free_ok = free_lanes;
    for (size_t j = 0; j < ps.items.size() && free_ok; ++j) free_ok = !dense[j] && __builtin_popcount(flips[j]) <= 1;
    if (free_ok) {
      std::vector<Segment> fr = memo_segments(e, flips, touch, dense, kk, R, true, lowb);
      if (segment_plan_cost(fr, flips, lc, xc, lowb) < segment_plan_cost(*out, flips, lc, xc, lowb)) *out = std::move(fr);
    }
    std::vector<uint32_t> ls;
    for (const Segment& sg : *out) {
      ls.push_back(sg.lanemask);
      L.free_lanes_used = L.free_lanes_used || sg.lanemask != 31u;
    }
    *swz = choose_swizzle(ls, kk);
    *outp = chosen;
    if (e->choice_memo.size() > 16384) e->choice_memo.clear();
    e->choice_memo.emplace(ck, std::make_pair(*outp, *swz));
  };
  if (L.reg) {
    // register-op units per amplitude: a lane flip is a warp shuffle of both (fwd:
    // one) buffers (4 SHFL per 16-byte amplitude at half the DFMA rate), a layout
    // change 32 B of shared-memory traffic per amplitude and buffer
    const double lc = kLaneCost, xc = kXposeCost;
    for (size_t si = 0; si < steps.size(); ++si)
      if (!steps[si].swap) pass_segments(steps[si].pass, pgates[si], pshapes[si], L.k, RB, lc, xc, &psegs[si], &pswz[si]);
    for (size_t si = 0; si < fsteps.size(); ++si)
      if (!fsteps[si].swap)
        pass_segments(fsteps[si].pass, fpgates[si], fpshapes[si], kf, RF, kFwdLaneCost, kFwdXposeCost, &psegs_f[si],
                      &pswz_f[si]);
  }
  auto reg_launch = [&](const Pass& ps, int nb, int kk) {
    Launch l;
    l.d = make_desc(nloc, kk, ps.qmask);
    l.kind = L_REG;
    l.nb = nb;
    l.R = nb == 1 ? RF : RB;
    l.threads = 32 << (kk - 5 - l.R);
    l.d.seg_begin = static_cast<int>(L.segs.size());
    l.d.op_begin = static_cast<int>(L.rops.size());  // this pass's register ops (staged in smem)
    return l;
  };
  auto swap_launch = [&](const Step& st) {
    Launch l;
    l.kind = L_SWAP;
    l.gbit = st.gbit;
    l.lpos = st.lpos;
    return l;
  };
  // default register layout for shared-memory segments: lowest non-lane positions
  auto default_regs = [](int R) { return ((1u << (5 + R)) - 1u) & ~31u; };

  // generated kernels keep the deferred scale C across layout changes (one
  // flush per tile, at the store) when a pass has no shared-memory segments
  const bool carry = jit_planned;
  auto all_reg = [](const std::vector<Segment>& v) {
    for (const Segment& sg : v)
      if (!sg.reg) return false;
    return true;
  };

  SVGB_PHASE(3);
  // forward schedule
  for (size_t si = 0; si < fsteps.size(); ++si) {
    if (fsteps[si].swap) {
      L.fwd.push_back(swap_launch(fsteps[si]));
      L.swap_bytes += S;  // half a shard out, half in
      continue;
    }
    const Pass& ps = fsteps[si].pass;
    const GateList& gs = fpgates[si];
    const TileMap tm = tile_map(ps.qmask);
    if (!L.reg) {
      Launch l;
      l.d = make_desc(nloc, L.k, ps.qmask);
      l.kind = L_SMEM_FWD;
      l.d.op_begin = static_cast<int>(L.ops.size());
      for (const svg_gate& gt : gs) emit_op(L, tm, gt, OP_APPLY_PAULI, 0, gt.fwd, 0);
      l.d.op_end = static_cast<int>(L.ops.size());
      L.fwd.push_back(l);
    } else {
      Launch l = reg_launch(ps, 1, kf);
      l.swz = pswz_f[si];
      uint32_t prev = ~0u, prev_l = ~0u;
      double C = 1.0;  // deferred scale; flushed when the layout changes (see SegDesc.scale)
      for (const Segment& sg : *psegs_f[si]) {
        SegLocal sl;
        SegDesc sd = make_seg(sg.reg ? SEG_REG : SEG_SMEM, sg.reg ? sg.regmask : default_regs(RF),
                              sg.reg ? sg.lanemask : 31u, l.swz, kf, RF, &sl);
        sd.same_map = sg.reg && sg.regmask == prev && sg.lanemask == prev_l;
        prev = sg.reg ? sg.regmask : ~0u;
        prev_l = sg.reg ? sg.lanemask : ~0u;
        if (!sd.same_map && !(carry && all_reg(*psegs_f[si]))) C = 1.0;
        if (sg.reg) {
          sd.op_begin = static_cast<int>(L.rops.size());
          for (int it : sg.items) emit_rop(L, tm, sl, gs[it], ROP_FWD, gs[it].fwd, nullptr, 0, real_sums, &C);
          sd.op_end = static_cast<int>(L.rops.size());
          sd.scale = C;
        } else {
          sd.op_begin = static_cast<int>(L.ops.size());
          for (int it : sg.items) emit_op(L, tm, gs[it], OP_APPLY_PAULI, 0, gs[it].fwd, 0);
          sd.op_end = static_cast<int>(L.ops.size());
          l.tiles = true;
        }
        L.segs.push_back(sd);
      }
      if (prev_l != ~0u && (prev_l & lowmask) != lowmask) {  // back to the global lane layout for the store
        SegLocal sl;
        SegDesc sd = make_seg(SEG_REG, default_regs(RF), 31u, l.swz, kf, RF, &sl);
        sd.op_begin = sd.op_end = static_cast<int>(L.rops.size());
        sd.scale = carry ? C : 1.0;
        L.segs.push_back(sd);
        l.tiles = true;
      }
      l.d.seg_end = static_cast<int>(L.segs.size());
      l.d.op_end = static_cast<int>(L.rops.size());
      if (psegs_f[si]->size() > 1) l.tiles = true;
      L.fwd.push_back(l);
    }
    L.pass_bytes += 2 * S;
  }

  // Early forward launches: generated kernels with register segments only need
  // no device tables (their coefficients travel in the launch parameters).
  if (fwd_ready && jit_planned && !e->jit_dry_run && !L.fwd.empty()) {
    bool ok = true;
    for (const Launch& l : L.fwd) {
      ok = ok && l.kind == L_REG;
      for (int si = l.d.seg_begin; ok && si < l.d.seg_end; ++si) ok = L.segs[si].kind == SEG_REG;
    }
    if (ok) {
      std::vector<JitPass> passes;
      for (Launch& l : L.fwd) {
        JitPass jp;
        jp.R = l.R;
        jp.nb = 1;
        jp.k = l.d.k;
        jp.nloc = nloc;
        jp.threads = l.threads;
        jp.tiles = l.tiles;
        jp.rest = l.d.rest;
        jp.q = l.d.q;
        jp.swz = l.swz.col;
        jp.scale_carry = carry;
        jp.checked = e->opt_checked != 0;
        jp.lowb = std::min(5, L.b);
        jp.segs = L.segs.data() + l.d.seg_begin;
        jp.nsegs = l.d.seg_end - l.d.seg_begin;
        jp.rops = L.rops.data() + l.d.op_begin;
        jp.op_begin = l.d.op_begin;
        passes.push_back(jp);
      }
      std::vector<std::shared_ptr<JitKernel>> ks;
      try {
        ks = jit_get(passes, e->device);
      } catch (const std::exception& ex) {
        throw JitFailure(ex.what());
      }
      for (size_t i = 0; i < ks.size(); ++i) {
        Launch& l = L.fwd[i];
        l.jit = ks[i];
        l.smem = l.jit->smem;
        if (l.jit->blocks_per_sm <= 0) {
          int blocks = 0;
          if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, reinterpret_cast<const void*>(l.jit->fn),
                                                            l.threads, l.smem) != cudaSuccess || blocks < 1) {
            (void)cudaGetLastError();
            blocks = 1;
          }
          l.jit->blocks_per_sm = blocks;
        }
        const int64_t nt = int64_t(1) << (nloc - l.d.k);
        l.grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nt, int64_t(e->sms) * l.jit->blocks_per_sm)));
      }
      fwd_ready(L);
      L.fwd_early = true;
    }
  }

  SVGB_PHASE(4);
  // observable passes keep 11-qubit tiles next to 12-qubit gate passes (their
  // per-term work is light: more, smaller tiles balance better -- measured cfg 3;
  // cfg 4: 45 / 56 / 93 ms at 11 / 12 / 13 tile qubits, although 13 saves a pass)
  PlanParams pp_obs = pp;
  if (jit_planned && L.k == 12 && e->opt_tile == 0) pp_obs.k = 11;
  const int kobs = pp_obs.k;
  // observable passes: terms in the final physical layout, grouped by the flip
  // pattern on rank bits (a nonzero pattern reads the partner shard's psi), then
  // by local flip mask into tiles
  const uint64_t loc_mask = (nloc >= 64) ? ~0ull : ((1ull << nloc) - 1);
  std::vector<uint64_t> xg_order;
  std::vector<std::vector<int>> by_xg;
  std::vector<svg_pauli_term> pterms(p->num_terms);
  for (int t = 0; t < p->num_terms; ++t) {
    pterms[t] = p->terms[t];
    pterms[t].x_mask = remap_mask(p->terms[t].x_mask, l2p_final);
    pterms[t].z_mask = remap_mask(p->terms[t].z_mask, l2p_final);
    const uint64_t xg = pterms[t].x_mask & ~loc_mask;
    size_t j = 0;
    while (j < xg_order.size() && xg_order[j] != xg) ++j;
    if (j == xg_order.size()) {
      xg_order.push_back(xg);
      by_xg.emplace_back();
    }
    by_xg[j].push_back(t);
  }
  int64_t part = 0;
  const int64_t energy_off = 0;
  for (size_t gidx = 0; gidx < xg_order.size(); ++gidx) {
    const uint64_t xg = xg_order[gidx];
    const std::vector<int>& members = by_xg[gidx];
    std::vector<uint64_t> flips(members.size());
    for (size_t j = 0; j < members.size(); ++j) flips[j] = pterms[members[j]].x_mask & loc_mask;
    std::vector<int> direct;
    std::vector<Pass> tpasses = plan_term_passes(flips, pp_obs, &direct);
    if (!direct.empty()) {  // wide flip masks: one untiled gather pass (qmask 0)
      Pass ps;
      ps.items = direct;
      tpasses.push_back(ps);
    }
    if (xg) L.obs.push_back(Launch{});  // exchange step: fetch the partner shard's psi
    if (xg) {
      L.obs.back().kind = L_FETCH;
      L.obs.back().d.xglob = xg;
      L.swap_bytes += 2 * S;
    }
    for (const Pass& ps : tpasses) {
      const TileMap tm = tile_map(ps.qmask);
      Launch l;
      l.d = make_desc(nloc, kobs, ps.qmask);
      l.d.op_begin = static_cast<int>(L.terms.size());
      l.d.untiled = ps.qmask == 0;
      l.d.xglob = xg;
      l.kind = l.d.untiled ? L_OBS_DIRECT : L_OBS;
      for (int ti : ps.items) {
        const svg_pauli_term& src = pterms[members[ti]];
        DevTerm dt;
        dt.c = cm(d2(src.coeff), ipow(src.n_y));
        const uint64_t xl = src.x_mask & loc_mask;
        if (l.d.untiled) {  // local flip mask split over (xl, zl); full z in zo
          dt.xl = static_cast<uint32_t>(xl);
          dt.zl = static_cast<uint32_t>(xl >> 32);
          dt.zo = src.z_mask;
        } else {
          dt.xl = tm.local(xl);
          dt.zl = tm.local(src.z_mask);
          dt.zo = src.z_mask & ~tm.qmask;
        }
        L.terms.push_back(dt);
      }
      if (!l.d.untiled)  // group equal flip masks (the kernel shares the partner amplitude)
        std::stable_sort(L.terms.begin() + l.d.op_begin, L.terms.end(),
                         [](const DevTerm& x, const DevTerm& y) { return x.xl < y.xl; });
      l.d.op_end = static_cast<int>(L.terms.size());
      l.d.accumulate = L.obs_kernels > 0;
      L.obs_kernels++;
      L.obs.push_back(l);
      L.pass_bytes += (l.d.accumulate ? 3 : 2) * S;
    }
  }

  // Product terms (factors kept as 2x2 matrices, e.g. hadamard_all): per term a
  // pipeline of tile passes, each applying the factors on its tile qubits; the
  // last pass accumulates coeff * (x)F psi into lambda with the energy partial.
  // Factors on rank bits (sharded states) are written in the Pauli basis
  // (F = aI + bX + cY + dZ): every rank flip pattern is a sub-pipeline reading
  // the partner shard, and the Z parts fold into a per-shard scalar.
  for (int t = 0; t < p->num_product_terms; ++t) {
    const svg_product_term& pt = p->product_terms[t];
    std::vector<std::pair<int, const svg_c128*>> locf;
    // rank-bit part: (x pattern, z pattern, weight), expanded factor by factor
    std::vector<std::tuple<uint64_t, uint64_t, double2>> subs = {{0ull, 0ull, make_double2(1.0, 0.0)}};
    for (int f = pt.first_factor; f < pt.first_factor + pt.num_factors; ++f) {
      const int q = l2p_final.empty() ? p->factors[f].qubit : l2p_final[p->factors[f].qubit];
      const svg_c128* m = p->factors[f].m;
      if (q < nloc) {
        locf.push_back({q, m});
        continue;
      }
      const uint64_t bit = 1ull << q;
      const double2 m0 = d2(m[0]), m1 = d2(m[1]), m2 = d2(m[2]), m3 = d2(m[3]);
      // F = a I + b X + c Y + d Z; c Y with Y = i^1 (-1)^{((m^x)&z)} X-flip: weight c*i
      const double2 a = make_double2(0.5 * (m0.x + m3.x), 0.5 * (m0.y + m3.y));
      const double2 dz = make_double2(0.5 * (m0.x - m3.x), 0.5 * (m0.y - m3.y));
      const double2 bx = make_double2(0.5 * (m1.x + m2.x), 0.5 * (m1.y + m2.y));
      const double2 cy = make_double2(-0.5 * (m1.y - m2.y), 0.5 * (m1.x - m2.x));  // i (m01 - m10) / 2
      const std::tuple<uint64_t, uint64_t, double2> parts[4] = {
          {0ull, 0ull, a}, {bit, 0ull, bx}, {bit, bit, cm(cy, make_double2(0.0, 1.0))}, {0ull, bit, dz}};
      std::vector<std::tuple<uint64_t, uint64_t, double2>> next;
      for (const auto& sb : subs)
        for (const auto& pa : parts) {
          const double2 w = cm(std::get<2>(sb), std::get<2>(pa));
          if (w.x == 0.0 && w.y == 0.0) continue;
          next.push_back({std::get<0>(sb) | std::get<0>(pa), std::get<1>(sb) | std::get<1>(pa), w});
        }
      subs.swap(next);
    }
    std::sort(locf.begin(), locf.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    // tile passes over the local factor qubits: the forced low qubits plus up to
    // kobs - b further factor qubits each (filled up with the lowest free qubits)
    const uint64_t low = (L.b >= 64) ? ~0ull : ((1ull << L.b) - 1);
    std::vector<std::vector<std::pair<int, const svg_c128*>>> chunks(1);
    int wide = 0;
    for (const auto& fq : locf) {
      if ((low >> fq.first) & 1) {
        chunks[0].push_back(fq);
        continue;
      }
      if (wide == kobs - L.b || int(chunks.back().size()) >= kMaxProdFactors) {
        chunks.emplace_back();
        wide = 0;
      }
      chunks.back().push_back(fq);
      ++wide;
    }
    // low-qubit factors ride in the first pass (chunk 0 may also hold wide ones)
    std::map<uint64_t, std::vector<std::pair<uint64_t, double2>>> by_x;
    for (const auto& sb : subs) by_x[std::get<0>(sb)].push_back({std::get<1>(sb), std::get<2>(sb)});
    for (const auto& xz : by_x) {
      const uint64_t xg = xz.first;
      if (xg) {
        L.obs.push_back(Launch{});
        L.obs.back().kind = L_FETCH;
        L.obs.back().d.xglob = xg;
        L.swap_bytes += 2 * S;
      }
      for (size_t c = 0; c < chunks.size(); ++c) {
        uint64_t qm = low;
        for (const auto& fq : chunks[c]) qm |= 1ull << fq.first;
        for (int q = 0; q < nloc && __builtin_popcountll(qm) < std::min(kobs, nloc); ++q) qm |= 1ull << q;
        Launch l;
        l.kind = L_PROD;
        l.d = make_desc(nloc, __builtin_popcountll(qm), qm);
        l.d.xglob = xg;
        const TileMap tm = tile_map(qm);
        l.prod.n = static_cast<int32_t>(chunks[c].size());
        for (size_t j = 0; j < chunks[c].size(); ++j) {
          l.prod.pos[j] = static_cast<uint32_t>(tm.pos[chunks[c][j].first]);
          for (int r = 0; r < 4; ++r) l.prod.m[j][r] = d2(chunks[c][j].second[r]);
        }
        l.prod_first = c == 0;
        l.prod.last = c + 1 == chunks.size();
        if (l.prod.last) {
          l.prod_coeff = d2(pt.coeff);
          l.prod_z = xz.second;
          l.d.accumulate = L.obs_kernels > 0;
          L.obs_kernels++;
          L.pass_bytes += (l.d.accumulate ? 4 : 3) * S;
        } else {
          L.pass_bytes += 2 * S;
        }
        L.obs.push_back(l);
      }
    }
  }

  SVGB_PHASE(5);
  // reverse schedule: steps backwards (swaps undo themselves on phi and lambda),
  // gates backwards inside each pass
  std::vector<std::pair<int, int>> deriv_slot(p->num_derivs, {-1, -1});  // (rev launch, slot)
  auto smem_reverse_ops = [&](const TileMap& tm, const svg_gate& gt, int gi, uint32_t& slot) {
    emit_op(L, tm, gt, OP_APPLY_PAULI, 0, gt.rewind, 0);
    for (int j = 0; j < gt.nderiv; ++j) {
      const int d = first_deriv[gi] + j;
      deriv_slot[d] = {static_cast<int>(L.rev.size()), static_cast<int>(slot)};
      emit_op(L, tm, gt, OP_IP_PAULI, 0, gens[d].pre, slot++);
    }
    if (gi > 0) emit_op(L, tm, gt, OP_APPLY_PAULI, 1, gt.adjoint, 0);
  };
  if (with_reverse) {
    for (int si = static_cast<int>(steps.size()) - 1; si >= 0; --si) {
      if (steps[si].swap) {
        L.rev.push_back(swap_launch(steps[si]));
        L.swap_bytes += 2 * S;
        continue;
      }
      const Pass& ps = steps[si].pass;
      const GateList& gs = pgates[si];
      const TileMap tm = tile_map(ps.qmask);
      uint32_t slot = 0;
      if (!L.reg) {
        Launch l;
        l.d = make_desc(nloc, L.k, ps.qmask);
        l.kind = L_SMEM_REV;
        l.d.op_begin = static_cast<int>(L.ops.size());
        for (int j = static_cast<int>(ps.items.size()) - 1; j >= 0; --j) smem_reverse_ops(tm, gs[j], ps.items[j], slot);
        l.d.op_end = static_cast<int>(L.ops.size());
        l.d.nslots = static_cast<int>(slot);
        L.rev.push_back(l);
      } else {
        Launch l = reg_launch(ps, 2, L.k);
        l.swz = pswz[si];
        const std::vector<Segment>& sgs = *psegs[si];
        uint32_t prev = ~0u, prev_l = ~0u;
        double C = 1.0;
        for (auto st = sgs.rbegin(); st != sgs.rend(); ++st) {
          const Segment& sg = *st;
          SegLocal sl;
          SegDesc sd = make_seg(sg.reg ? SEG_REG : SEG_SMEM, sg.reg ? sg.regmask : default_regs(RB),
                                sg.reg ? sg.lanemask : 31u, l.swz, L.k, RB, &sl);
          sd.same_map = sg.reg && sg.regmask == prev && sg.lanemask == prev_l;
          prev = sg.reg ? sg.regmask : ~0u;
          prev_l = sg.reg ? sg.lanemask : ~0u;
          if (!sd.same_map && !(carry && all_reg(sgs))) C = 1.0;
          if (sg.reg) {
            sd.op_begin = static_cast<int>(L.rops.size());
            for (auto it = sg.items.rbegin(); it != sg.items.rend(); ++it) {
              const int gi = ps.items[*it];
              const svg_gate& gt = gs[*it];
              const svg_c128* kpost = nullptr;
              if (gt.nderiv == 1) {
                const int d = first_deriv[gi];
                deriv_slot[d] = {static_cast<int>(L.rev.size()), static_cast<int>(slot)};
                kpost = gens[d].post;
              }
              // one op rewinds phi AND lambda (rewind == adjoint for register-capable gates);
              // the reference skips lambda's update at i = 0, whose value is never read again
              emit_rop(L, tm, sl, gt, ROP_REV, gt.rewind, kpost, kpost ? slot++ : 0, real_sums, &C);
            }
            sd.op_end = static_cast<int>(L.rops.size());
            sd.scale = C;
          } else {
            sd.op_begin = static_cast<int>(L.ops.size());
            for (auto it = sg.items.rbegin(); it != sg.items.rend(); ++it)
              smem_reverse_ops(tm, gs[*it], ps.items[*it], slot);
            sd.op_end = static_cast<int>(L.ops.size());
            l.tiles = true;
          }
          L.segs.push_back(sd);
        }
        if (prev_l != ~0u && (prev_l & lowmask) != lowmask) {  // back to the global lane layout for the store
          SegLocal sl;
          SegDesc sd = make_seg(SEG_REG, default_regs(RB), 31u, l.swz, L.k, RB, &sl);
          sd.op_begin = sd.op_end = static_cast<int>(L.rops.size());
          sd.scale = carry ? C : 1.0;
          L.segs.push_back(sd);
          l.tiles = true;
        }
        l.d.seg_end = static_cast<int>(L.segs.size());
        l.d.op_end = static_cast<int>(L.rops.size());
        if (sgs.size() > 1) l.tiles = true;
        l.d.nslots = static_cast<int>(slot);
        L.rev.push_back(l);
      }
      L.pass_bytes += 4 * S;
    }
  }

  SVGB_PHASE(6);
  // grids, shared memory, partial offsets
  auto ntiles_of = [&](const Launch& l) {
    return int64_t(1) << (nloc - ((l.kind == L_REG || l.kind == L_OBS) ? l.d.k : L.k));
  };
  // lane-group inner-product accumulators: combine 2^shift lanes so that the
  // shared accumulators stay within 24 KB (two 128-thread CTAs with 64 KB of
  // transpose tiles still fit an SM; no per-op full warp reductions)
  const size_t acc_budget = size_t(24) << 10;
  auto set_thread_acc = [acc_budget](Launch& l) {
    l.d.thread_acc = l.nb == 2 && l.d.nslots > 0;
    l.d.acc_shift = 0;
    while (l.d.acc_shift < 5 && size_t(l.d.nslots) * (l.threads >> l.d.acc_shift) * sizeof(double) > acc_budget)
      ++l.d.acc_shift;
  };
  auto memo_occ = [&](int kind, int R, int threads, size_t smem, auto query) {
    const auto key = std::make_tuple(kind, R, threads, smem);
    auto it = e->occ_memo.find(key);
    if (it != e->occ_memo.end()) return it->second;
    const int v = query();
    e->occ_memo[key] = v;
    return v;
  };
  auto clamp_grid_k = [&](int per_sm, int64_t ntiles) {
    const int64_t slots = int64_t(e->sms) * per_sm;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, slots)));
  };
  const int64_t ntiles_std = int64_t(1) << (nloc - L.k);
  auto clamp_grid = [&](int per_sm) { return clamp_grid_k(per_sm, ntiles_std); };
  auto size_launch = [&](Launch& l) {
    switch (l.kind) {
      case L_SMEM_FWD:
        l.smem = fwd_smem(L.k, l.d.b);
        l.grid = clamp_grid(memo_occ(-1, 0, 0, l.smem, [&] { return occupancy(0, l.smem); }));
        break;
      case L_SMEM_REV:
        l.smem = rev_smem(L.k, l.d.b, l.d.nslots);
        l.grid = clamp_grid(memo_occ(-2, 0, 0, l.smem, [&] { return occupancy(2, l.smem); }));
        break;
      case L_REG:
        // per-thread inner-product accumulators when they fit a modest budget
        set_thread_acc(l);
        if (l.jit) {
          l.smem = l.jit->smem;
          if (l.jit->blocks_per_sm <= 0) {
            int blocks = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, reinterpret_cast<const void*>(l.jit->fn),
                                                              l.threads, l.smem) != cudaSuccess || blocks < 1) {
              (void)cudaGetLastError();
              blocks = 1;
            }
            l.jit->blocks_per_sm = blocks;
          }
          l.grid = clamp_grid_k(l.jit->blocks_per_sm, ntiles_of(l));
          break;
        }
        l.smem = reg_smem(L.k, l.nb, l.threads / 32, l.d.nslots, l.d.op_end - l.d.op_begin,
                          l.d.seg_end - l.d.seg_begin, l.tiles, l.d.thread_acc != 0, l.d.acc_shift);
        l.grid = clamp_grid(memo_occ(l.nb, l.R, l.threads, l.smem, [&] { return reg_occupancy(l.nb, l.R, l.threads, l.smem); }));
        break;
      case L_OBS:
        if (l.jit) {
          l.smem = l.jit->smem;
          if (l.jit->blocks_per_sm <= 0) {
            int blocks = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, reinterpret_cast<const void*>(l.jit->fn),
                                                              kThreads, l.smem) != cudaSuccess || blocks < 1) {
              (void)cudaGetLastError();
              blocks = 1;
            }
            l.jit->blocks_per_sm = blocks;
          }
          l.grid = clamp_grid_k(l.jit->blocks_per_sm, ntiles_of(l));
          break;
        }
        l.smem = obs_smem(l.d.k, l.d.b, l.d.op_end - l.d.op_begin);
        l.grid = clamp_grid_k(memo_occ(-3, 0, 0, l.smem, [&] { return occupancy(1, l.smem); }), ntiles_of(l));
        break;
      case L_PROD:
        l.smem = prod_smem(l.d.k, l.d.b);
        l.grid = clamp_grid_k(memo_occ(-4, l.d.k, 0, l.smem, [&] { return occupancy(3, l.smem); }), ntiles_of(l));
        break;
      case L_OBS_DIRECT:
        l.smem = 0;
        l.grid = std::max(1, static_cast<int>(std::min<int64_t>(int64_t(e->sms) * 8, int64_t(1) << std::max(0, nloc - 8))));
        break;
      default:  // exchanges: no kernel grid of their own
        l.smem = 0;
        l.grid = 0;
    }
    if (l.smem > e->max_smem) throw InvalidArg("pass needs more shared memory than the device offers");
  };
  SVGB_PHASE(7);
  // circuit-specialised kernels for the register-tile passes
  const bool want_jit = L.reg && (e->opt_jit == 2 || (e->opt_jit == 1 && nloc >= kJitMinQubits));
  if (want_jit) {
    std::vector<Launch*> regl;
    for (std::vector<Launch>* v : {&L.fwd, &L.rev})
      for (Launch& l : *v)
        if (l.kind == L_REG && !l.jit) regl.push_back(&l);
    std::vector<JitPass> passes;
    passes.reserve(regl.size());
    for (Launch* l : regl) {
      set_thread_acc(*l);
      if (l->d.thread_acc) {
        // auto budget: the SM's shared memory split over the kernel's CTAs per SM,
        // minus tile / staging buffers and per-warp accumulators.  Every halving
        // of the accumulators costs a butterfly step per op (measured: 40-slot
        // passes 8 % slower at shift 1 than at shift 0).
        const int blocks = l->nb == 2 ? std::max(1, std::min(2, 256 / l->threads)) : (l->R == 3 ? 2 : 4);
        const size_t share = std::min<size_t>(e->max_smem, (size_t(e->max_smem_sm) / blocks) - 1024);
        const size_t fixed = (sizeof(double2) << l->d.k) * l->nb + sizeof(double2) * (l->threads / 32) * l->d.nslots;
        const size_t budget = share > fixed + 4096 ? share - fixed : 4096;
        l->d.acc_shift = 0;
        while (l->d.acc_shift < 5 && size_t(l->d.nslots) * (l->threads >> l->d.acc_shift) * sizeof(double) > budget)
          ++l->d.acc_shift;
      }
      JitPass jp;
      jp.R = l->R;
      jp.nb = l->nb;
      jp.k = l->d.k;
      jp.nloc = nloc;
      jp.threads = l->threads;
      jp.nslots = l->d.nslots;
      jp.thread_acc = l->d.thread_acc != 0;
      jp.acc_shift = l->d.acc_shift;
      jp.tiles = l->tiles;
      jp.rest = l->d.rest;
      jp.q = l->d.q;
      jp.swz = l->swz.col;
      jp.scale_carry = carry;
      jp.checked = e->opt_checked != 0;
      jp.lowb = std::min(5, L.b);
      jp.segs = L.segs.data() + l->d.seg_begin;
      jp.nsegs = l->d.seg_end - l->d.seg_begin;
      jp.rops = L.rops.data() + l->d.op_begin;
      jp.op_begin = l->d.op_begin;
      passes.push_back(jp);
    }
    try {
      if (e->jit_dry_run == 2) {  // svg_debug_plan_stats: the plan's shape, nothing generated
        double* st = e->plan_stats;
        for (const Launch* l : regl) {
          const int o = l->nb == 2 ? 8 : 0;
          st[o + 0] += 1;  // passes
          for (int si = l->d.seg_begin; si < l->d.seg_end; ++si) {
            const SegDesc& sg = L.segs[si];
            st[o + 1] += 1;                                                      // segments
            if (std::getenv("SVGB_PLAN_DUMP") && sg.kind == SEG_REG) {
              std::fprintf(stderr, "%s pass %d seg %d ops %d same %d lanes", l->nb == 2 ? "rev" : "fwd", int(st[o + 0]),
                           si - l->d.seg_begin, sg.op_end - sg.op_begin, int(sg.same_map));
              for (int i = 0; i < 5; ++i) std::fprintf(stderr, " %d", int(l->d.q[sg.lanepos[i]]));
              std::fprintf(stderr, " | regs");
              for (int i = 0; i < l->R; ++i) std::fprintf(stderr, " %d", int(l->d.q[sg.regpos[i]]));
              std::fprintf(stderr, " | warps");
              for (int i = 0; i < l->d.k - 5 - l->R; ++i) std::fprintf(stderr, " %d", int(l->d.q[sg.warppos[i]]));
              std::fprintf(stderr, "\n");
            }
            if (si > l->d.seg_begin && !(sg.kind == SEG_REG && sg.same_map)) st[o + 2] += 1;  // layout changes
            if (si > l->d.seg_begin && sg.kind == SEG_REG && !sg.same_map && L.segs[si - 1].kind == SEG_REG) {
              // layout changes that exchange m register positions with warp positions, all else in place
              const SegDesc& pv = L.segs[si - 1];
              const int wb = l->d.k - 5 - l->R;
              bool ok = std::memcmp(pv.lanepos, sg.lanepos, 5) == 0;
              int m = 0;
              for (int i = 0; i < wb && ok; ++i) {
                if (pv.warppos[i] == sg.warppos[i]) continue;
                ++m;
                bool a = false, b = false;
                for (int r = 0; r < l->R; ++r) {
                  a = a || sg.regpos[r] == pv.warppos[i];
                  b = b || pv.regpos[r] == sg.warppos[i];
                }
                ok = a && b;
              }
              if (ok && m == 1) st[o + 7] += 1;
              if (ok && m == 2) st[o + 6] += 0;  // (not counted)
            }
            if (sg.kind != SEG_REG) continue;
            for (int oi = sg.op_begin; oi < sg.op_end; ++oi) {
              st[o + 3] += 1;                                                    // register ops
              if (L.rops[oi].xl) st[o + 4] += 1;                                 // lane flips
            }
          }
          st[o + 5] = std::max(st[o + 5], double(l->d.nslots));
          if (l->d.acc_shift) st[o + 6] += 1;                                    // passes with lane-group accumulators
        }
        throw std::runtime_error("dry run");
      }
      std::string why;
      if (!jit_available(&why)) throw std::runtime_error(why);
      std::vector<std::shared_ptr<JitKernel>> ks = jit_get(passes, e->jit_dry_run ? -1 : e->device);
      for (size_t i = 0; i < ks.size(); ++i) regl[i]->jit = ks[i];
      // observable passes (tiled)
      std::vector<Launch*> obsl;
      std::vector<JitObsPass> opasses;
      for (Launch& l : L.obs) {
        if (l.kind != L_OBS) continue;
        JitObsPass op;
        op.k = l.d.k;
        op.b = l.d.b;
        op.nloc = nloc;
        op.threads = kThreads;
        op.rest = l.d.rest;
        op.q = l.d.q;
        op.terms = L.terms.data() + l.d.op_begin;
        op.nterms = l.d.op_end - l.d.op_begin;
        op.accumulate = l.d.accumulate != 0;
        op.remote = l.d.xglob != 0;
        obsl.push_back(&l);
        opasses.push_back(op);
      }
      std::vector<std::shared_ptr<JitKernel>> ko = jit_get_obs(opasses, e->jit_dry_run ? -1 : e->device);
      for (size_t i = 0; i < ko.size(); ++i) obsl[i]->jit = ko[i];
      if (e->jit_dry_run) {  // svg_debug_jit_check: sources generated and compiled; keep the interpreter
        e->jit_dry_count += static_cast<int>(passes.size() + opasses.size());
        throw std::runtime_error("dry run");
      }
    } catch (const std::exception& ex) {
      if (e->jit_dry_run && std::string(ex.what()) != "dry run") throw;
      // plans made for the generated kernels (free lanes, carried scales, short
      // tile rows) cannot run on the interpreter: the caller re-lowers
      if ((e->opt_jit == 2 || L.free_lanes_used || carry || L.b < 5) && !e->jit_dry_run) throw JitFailure(ex.what());
      e->jit_error = ex.what();  // auto: keep the interpreted kernels
    }
  }
  for (Launch& l : L.fwd) size_launch(l);
  for (Launch& l : L.obs) {
    size_launch(l);
    if (l.kind == L_FETCH) continue;
    l.d.part_off = part;
    part += l.grid;
  }
  const int64_t energy_count = part - energy_off;
  for (Launch& l : L.rev) {
    size_launch(l);
    if (l.kind == L_SWAP) continue;
    l.d.part_off = part;
    part += int64_t(l.d.nslots) * l.grid;
  }
  L.partial_count = part;
  if (with_reverse) {
    L.sums.resize(p->num_derivs + 1);
    for (int d = 0; d < p->num_derivs; ++d) {
      const Launch& l = L.rev[deriv_slot[d].first];
      L.sums[d] = SumSpec{l.d.part_off + int64_t(deriv_slot[d].second) * l.grid, l.grid};
    }
  } else {
    L.sums.resize(1);
  }
  L.sums.back() = SumSpec{energy_off, energy_count};
  for (const Step& st : steps) L.swaps += st.swap;
  SVGB_PHASE(8);
  return L;
}

struct Blob {
  size_t ops, coef, terms, sums, rops, segs, total;
};

Blob layout(const Lowered& L) {
  Blob b;
  size_t o = 0;
  b.ops = o;
  o = align_up(o + L.ops.size() * sizeof(DevOp), 256);
  b.coef = o;
  o = align_up(o + L.coef.size() * sizeof(double2), 256);
  b.terms = o;
  o = align_up(o + L.terms.size() * sizeof(DevTerm), 256);
  b.sums = o;
  o = align_up(o + L.sums.size() * sizeof(SumSpec), 256);
  b.rops = o;
  o = align_up(o + L.rops.size() * sizeof(RegOp), 256);
  b.segs = o;
  o = align_up(o + L.segs.size() * sizeof(SegDesc), 256);
  b.total = std::max<size_t>(o, 256);
  return b;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// One shard-local pass launch (sh: index of the shard held by this engine).
struct ShardView {
  double2* psi;
  double2* lam;
  double2* part;
  uint64_t rank_bits;
};

int run(svg_engine* e, const svg_problem* p, bool with_reverse, svg_c128* sums_out,
        svg_c128* deriv_out, svg_c128* energy_out, svg_stats* stats) {
  if (!e) return fail(SVG_EINVAL, "null engine");
  try {
    const auto t_enter = std::chrono::steady_clock::now();
    validate(p);
    if (e->shard_bits > 0 && e->shards_local == 1 && !e->comm)
      throw NcclError("the engine's NCCL communicator was aborted after an earlier failure");
    CK(cudaSetDevice(e->device));
    // A host input state starts its (large) host -> device copy before the host-side
    // lowering, which then overlaps the transfer; shards are consecutive slices of
    // the full index range (identity layout at the start).
    bool input_copied = false, chunked = false;
    if (p->input_amps) {
      const size_t amps0 = (size_t(1) << (p->num_qubits - e->shard_bits)) * e->shards_local;
      // SVG_FLAG_INPUT_LOCAL: the host array is this rank's slice only (no 2^n host copy per rank)
      const size_t first0 = (e->comm && !(p->flags & SVG_FLAG_INPUT_LOCAL))
                                ? size_t(e->rank) * (size_t(1) << (p->num_qubits - e->shard_bits)) : 0;
      e->psi.reserve(amps0 * sizeof(double2));
      // One shard of >= kChunkMinQubits qubits with generated kernels: the copy goes out
      // in kInputChunks chunks on its own stream, and the leading forward passes (those
      // whose tile qubits all lie below the chunk boundary) follow it chunk by chunk
      // (fwd_cb below) instead of waiting for the whole 16 * 2^n bytes.
      chunked = e->shards_local == 1 && !e->comm && e->opt_jit != 0 && p->num_qubits >= chunk_min_qubits();
      if (chunked) {
        if (!e->copy_stream) {
          CK(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
          CK(cudaEventCreateWithFlags(&e->enter_ev, cudaEventDisableTiming));
          for (cudaEvent_t& ev : e->chunk_ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        }
        CK(cudaEventRecord(e->ev[0], e->stream));  // the timed region starts with the copy
        CK(cudaEventRecord(e->enter_ev, e->stream));
        CK(cudaStreamWaitEvent(e->copy_stream, e->enter_ev, 0));
        const size_t camps = amps0 / svg_engine::kInputChunks;
        for (int c = 0; c < svg_engine::kInputChunks; ++c) {
          CK(cudaMemcpyAsync(static_cast<double2*>(e->psi.ptr) + c * camps, p->input_amps + c * camps,
                             camps * sizeof(double2), cudaMemcpyHostToDevice, e->copy_stream));
          CK(cudaEventRecord(e->chunk_ev[c], e->copy_stream));
        }
      } else {
        CK(cudaMemcpyAsync(e->psi.ptr, p->input_amps + first0, amps0 * sizeof(double2), cudaMemcpyHostToDevice,
                           e->stream));
      }
      input_copied = true;
    }
    // One shard: the initial state is set up before the lowering, and the forward
    // passes go out as soon as they are lowered (lower()'s fwd_ready), so the GPU
    // runs them while the host lowers the observable and the reverse sweep.
    const bool early = e->shards_local == 1 && !e->comm;
    int64_t early_launches = 0;
    std::function<void(Lowered&)> fwd_cb;
    if (early) {
      const size_t amps0 = size_t(1) << p->num_qubits;
      e->psi.reserve(amps0 * sizeof(double2));
      if (!chunked) CK(cudaEventRecord(e->ev[0], e->stream));
      if (!p->input_amps) {
        CK(cudaMemsetAsync(e->psi.ptr, 0, amps0 * sizeof(double2), e->stream));
        launch_set_basis(static_cast<double2*>(e->psi.ptr), static_cast<uint64_t>(p->input_basis), e->stream);
        ++early_launches;
      }
      if (!chunked) CK(cudaEventRecord(e->ev[1], e->stream));
      fwd_cb = [&](Lowered& Lf) {
        double2* psi0 = static_cast<double2*>(e->psi.ptr);
        const int nq = p->num_qubits;
        auto launch_range = [&](const Launch& l, uint64_t t0, uint64_t t1) {
          const JitArgsHead head{psi0, nullptr, nullptr, nullptr, nullptr, l.d.part_off, 0, t0, t1};
          std::vector<unsigned char> args =
              jit_args(*l.jit, head, Lf.segs.data() + l.d.seg_begin, Lf.rops.data() + l.d.op_begin);
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(static_cast<unsigned>(std::min<uint64_t>(l.grid, t1 - t0)));
          cfg.blockDim = dim3(l.threads);
          cfg.dynamicSmemBytes = l.smem;
          cfg.stream = e->stream;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          attr[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          void* params[] = {args.data()};
          CK(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(l.jit->fn), params));
          ++early_launches;
        };
        size_t lead = 0;  // leading passes whose tiles lie inside one input chunk
        if (chunked) {
          const int cq = nq - 4;  // log2(amplitudes per chunk); kInputChunks == 16
          while (lead < Lf.fwd.size()) {
            const PassDesc& d = Lf.fwd[lead].d;
            bool inside = true;
            for (int i = 0; i < d.k; ++i) inside = inside && d.q[i] < cq;
            if (!inside) break;
            ++lead;
          }
          for (int c = 0; c < svg_engine::kInputChunks; ++c) {
            CK(cudaStreamWaitEvent(e->stream, e->chunk_ev[c], 0));
            for (size_t i = 0; i < lead; ++i) {
              const uint64_t per = uint64_t(1) << (cq - Lf.fwd[i].d.k);  // tiles per chunk
              launch_range(Lf.fwd[i], c * per, (c + 1) * per);
            }
          }
          CK(cudaEventRecord(e->ev[1], e->stream));
        }
        for (size_t i = lead; i < Lf.fwd.size(); ++i)
          launch_range(Lf.fwd[i], 0, uint64_t(1) << (nq - Lf.fwd[i].d.k));
        CK(cudaEventRecord(e->ev[2], e->stream));
      };
    }
    bool init_done = early;  // psi initialised before the lowering (ev[0], ev[1] recorded)
    Lowered L;
    try {
      L = lower(e, p, with_reverse, fwd_cb);
    } catch (const JitFailure& ex) {
      if (e->opt_jit == 2) throw;
      // auto mode: generated kernels unavailable -- plan again for the interpreted
      // kernels; psi is set up again (early forward launches may have run)
      e->jit_error = ex.what();
      L = lower(e, p, with_reverse, {}, true);
      if (chunked) CK(cudaStreamWaitEvent(e->stream, e->chunk_ev[svg_engine::kInputChunks - 1], 0));
      chunked = false;
      init_done = false;
      input_copied = false;
    }
    if (chunked && !L.fwd_early) {  // no early forward launches: the stream waits for the whole copy
      CK(cudaStreamWaitEvent(e->stream, e->chunk_ev[svg_engine::kInputChunks - 1], 0));
      CK(cudaEventRecord(e->ev[1], e->stream));
    }
    const auto t_lowered = std::chrono::steady_clock::now();
    const int nloc = L.nloc;
    const int nsh = e->shards_local;       // shards held by this engine
    const size_t shard_amps = size_t(1) << nloc;
    const size_t amps = shard_amps * nsh;  // amplitudes held on this device
    const int64_t cnt = static_cast<int64_t>(L.sums.size());
    const int world = 1 << e->shard_bits;
    cudaStream_t s = e->stream;

    e->psi.reserve(amps * sizeof(double2));
    e->lam.reserve(amps * sizeof(double2));
    e->partials.reserve(std::max<int64_t>(1, L.partial_count) * nsh * sizeof(double2));
    const Blob bl = layout(L);
    e->blob.reserve(bl.total);
    e->hblob.reserve(bl.total);
    e->results.reserve(cnt * std::max(nsh, world) * sizeof(double2));
    e->hres.reserve(cnt * std::max(nsh, world) * sizeof(double2));
    const bool emulate = !e->comm && nsh > 1 && e->opt_emulate_transport;
    if (emulate) e->scratch.reserve(2 * shard_amps * sizeof(double2));
    bool multi_pass_products = false;  // a product pipeline of >= 2 passes keeps its tile in prodbuf
    for (const Launch& l : L.obs) multi_pass_products = multi_pass_products || (l.kind == L_PROD && !l.prod.last);
    if (multi_pass_products) e->prodbuf.reserve(amps * sizeof(double2));
    if (e->comm) {
      // exchange staging: one shard (partner fetch / one buffer's swap), two when the
      // reverse sweep swaps phi and lambda together
      bool rev_swaps = false;
      for (const Launch& l : L.rev) rev_swaps = rev_swaps || l.kind == L_SWAP;
      e->scratch.reserve((rev_swaps ? 2 : 1) * shard_amps * sizeof(double2));
      e->gathered.reserve(cnt * world * sizeof(double2));
    }

    char* hb = static_cast<char*>(e->hblob.ptr);
    char* db = static_cast<char*>(e->blob.ptr);
    // the pinned staging buffer may still feed a previous call's copy (its event;
    // a full stream sync would also wait for this call's early forward passes)
    if (e->blob_ev) CK(cudaEventSynchronize(e->blob_ev));
    std::memcpy(hb + bl.ops, L.ops.data(), L.ops.size() * sizeof(DevOp));
    std::memcpy(hb + bl.coef, L.coef.data(), L.coef.size() * sizeof(double2));
    std::memcpy(hb + bl.terms, L.terms.data(), L.terms.size() * sizeof(DevTerm));
    std::memcpy(hb + bl.sums, L.sums.data(), L.sums.size() * sizeof(SumSpec));
    std::memcpy(hb + bl.rops, L.rops.data(), L.rops.size() * sizeof(RegOp));
    std::memcpy(hb + bl.segs, L.segs.data(), L.segs.size() * sizeof(SegDesc));

    double2* psi = static_cast<double2*>(e->psi.ptr);
    double2* lam = static_cast<double2*>(e->lam.ptr);
    double2* part = static_cast<double2*>(e->partials.ptr);
    double2* scratch = static_cast<double2*>(e->scratch.ptr);
    const DevOp* dops = reinterpret_cast<const DevOp*>(db + bl.ops);
    const double2* dcoef = reinterpret_cast<const double2*>(db + bl.coef);
    const DevTerm* dterms = reinterpret_cast<const DevTerm*>(db + bl.terms);
    const SumSpec* dsums = reinterpret_cast<const SumSpec*>(db + bl.sums);
    const RegOp* drops = reinterpret_cast<const RegOp*>(db + bl.rops);
    const SegDesc* dsegs = reinterpret_cast<const SegDesc*>(db + bl.segs);
    double2* dres = static_cast<double2*>(e->results.ptr);

    auto view = [&](int sh) {
      const int rank = e->comm ? e->rank : sh;
      return ShardView{psi + sh * shard_amps, lam + sh * shard_amps, part + sh * std::max<int64_t>(1, L.partial_count),
                       uint64_t(rank) << nloc};
    };
    const Nccl* nccl = e->comm ? &Nccl::get() : nullptr;
    const size_t half_bytes = shard_amps / 2 * sizeof(double2);
    // rank bit `gbit` <-> local position `lpos` for one state buffer (see plan.h)
    auto swap_buffer = [&](double2* buf, int gbit, int lpos) {
      if (emulate) {  // every pair runs the rank-side pack / exchange / unpack sequence
        for (int r = 0; r < nsh; ++r) {
          if ((r >> gbit) & 1) continue;
          const int q = r | (1 << gbit);
          double2* sr = scratch;                  // r's outgoing half
          double2* sq = scratch + shard_amps / 2; // q's outgoing half
          launch_half_pack(buf + r * shard_amps, sr, nloc, lpos, 1, s);
          launch_half_pack(buf + q * shard_amps, sq, nloc, lpos, 0, s);
          launch_half_unpack(sq, buf + r * shard_amps, nloc, lpos, 1, s);
          launch_half_unpack(sr, buf + q * shard_amps, nloc, lpos, 0, s);
        }
        return;
      }
      if (!e->comm) {
        launch_swap_virtual(buf, nloc, nsh, gbit, lpos, s);
        return;
      }
      const int a = (e->rank >> gbit) & 1, partner = e->rank ^ (1 << gbit);
      double2* send = scratch;
      double2* recv = scratch + shard_amps / 2;
      launch_half_pack(buf, send, nloc, lpos, 1 - a, s);
      nccl->check(nccl->group_start(), "ncclGroupStart");
      nccl->check(nccl->send(send, half_bytes, kNcclUint8, partner, e->comm, s), "ncclSend");
      nccl->check(nccl->recv(recv, half_bytes, kNcclUint8, partner, e->comm, s), "ncclRecv");
      nccl->check(nccl->group_end(), "ncclGroupEnd");
      launch_half_unpack(recv, buf, nloc, lpos, 1 - a, s);
    };
    // reverse-sweep swaps exchange phi AND lambda: over NCCL both halves go out in
    // one group (two concurrent transfers per partner instead of two back-to-back
    // exchanges); scratch holds [phi send | phi recv | lambda send | lambda recv]
    auto swap_pair = [&](int gbit, int lpos) {
      if (!e->comm) {
        swap_buffer(psi, gbit, lpos);
        swap_buffer(lam, gbit, lpos);
        return;
      }
      const int a = (e->rank >> gbit) & 1, partner = e->rank ^ (1 << gbit);
      const size_t h = shard_amps / 2;
      launch_half_pack(psi, scratch, nloc, lpos, 1 - a, s);
      launch_half_pack(lam, scratch + 2 * h, nloc, lpos, 1 - a, s);
      nccl->check(nccl->group_start(), "ncclGroupStart");
      nccl->check(nccl->send(scratch, half_bytes, kNcclUint8, partner, e->comm, s), "ncclSend");
      nccl->check(nccl->recv(scratch + h, half_bytes, kNcclUint8, partner, e->comm, s), "ncclRecv");
      nccl->check(nccl->send(scratch + 2 * h, half_bytes, kNcclUint8, partner, e->comm, s), "ncclSend");
      nccl->check(nccl->recv(scratch + 3 * h, half_bytes, kNcclUint8, partner, e->comm, s), "ncclRecv");
      nccl->check(nccl->group_end(), "ncclGroupEnd");
      launch_half_unpack(scratch + h, psi, nloc, lpos, 1 - a, s);
      launch_half_unpack(scratch + 3 * h, lam, nloc, lpos, 1 - a, s);
    };
    auto fetch_partner = [&](uint64_t xglob) {  // partner shard's psi -> scratch (NCCL mode)
      const int partner = e->rank ^ static_cast<int>(xglob >> nloc);
      nccl->check(nccl->group_start(), "ncclGroupStart");
      nccl->check(nccl->send(psi, shard_amps * sizeof(double2), kNcclUint8, partner, e->comm, s), "ncclSend");
      nccl->check(nccl->recv(scratch, shard_amps * sizeof(double2), kNcclUint8, partner, e->comm, s), "ncclRecv");
      nccl->check(nccl->group_end(), "ncclGroupEnd");
    };

    int jit_launches = 0;
    // generated kernels go out with programmatic dependent launch (they call
    // griddepcontrol.wait before their first global access)
    auto launch_generated = [&](cudaKernel_t fn, int grid, int threads, size_t smem, cudaStream_t st,
                                std::vector<unsigned char>& args) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      void* params[] = {args.data()};
      CK(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(fn), params));
    };
    // register-tile pass: the circuit-specialised kernel when there is one, else the interpreter
    auto launch_reg = [&](const Launch& l, const PassDesc& d, double2* b0, double2* b1, double2* prt) {
      if (!l.jit) {
        launch_pass_reg(l.nb, l.R, d, l.grid, l.threads, l.smem, s, b0, b1, dsegs, drops, dops, dcoef, prt);
        return;
      }
      const JitArgsHead head{b0, b1, dops, dcoef, prt, d.part_off, d.rank_bits, 0, uint64_t(1) << (nloc - d.k)};
      std::vector<unsigned char> args =
          jit_args(*l.jit, head, L.segs.data() + d.seg_begin, L.rops.data() + d.op_begin);
      launch_generated(l.jit->fn, l.grid, l.threads, l.smem, s, args);
      ++jit_launches;
    };
    int64_t launches = 0, h2d = bl.total, d2h = 0;
    const auto t_launch = std::chrono::steady_clock::now();
    if (!init_done) CK(cudaEventRecord(e->ev[0], s));
    CK(cudaMemcpyAsync(db, hb, bl.total, cudaMemcpyHostToDevice, s));
    if (!e->blob_ev) CK(cudaEventCreateWithFlags(&e->blob_ev, cudaEventDisableTiming));
    CK(cudaEventRecord(e->blob_ev, s));
    // input: shards are consecutive slices of the full index range (identity layout at the start)
    const size_t first_amp = e->comm ? size_t(e->rank) * shard_amps : 0;
    if (p->input_amps) {
      const size_t src_off = (p->flags & SVG_FLAG_INPUT_LOCAL) ? 0 : first_amp;
      if (!input_copied)
        CK(cudaMemcpyAsync(psi, p->input_amps + src_off, amps * sizeof(double2), cudaMemcpyHostToDevice, s));
      h2d += amps * sizeof(double2);
    } else if (!init_done) {
      CK(cudaMemsetAsync(psi, 0, amps * sizeof(double2), s));
      const uint64_t idx = static_cast<uint64_t>(p->input_basis);
      if (idx >= first_amp && idx < first_amp + amps) {
        launch_set_basis(psi, idx - first_amp, s);
        launches += 1;
      }
    }
    launches += early_launches;
    if (!init_done) CK(cudaEventRecord(e->ev[1], s));
    for (const Launch& l : L.fwd) {
      if (L.fwd_early) break;  // launched by the fwd_ready callback
      if (l.kind == L_SWAP) {
        swap_buffer(psi, l.gbit, l.lpos);
        continue;
      }
      for (int sh = 0; sh < nsh; ++sh) {
        const ShardView v = view(sh);
        PassDesc d = l.d;
        d.rank_bits = v.rank_bits;
        if (l.kind == L_REG)
          launch_reg(l, d, v.psi, nullptr, v.part);
        else
          launch_fwd(d, l.grid, l.smem, s, v.psi, dops, dcoef);
        ++launches;
      }
    }
    if (!L.fwd_early) CK(cudaEventRecord(e->ev[2], s));
    double2* prodbuf = static_cast<double2*>(e->prodbuf.ptr);
    for (const Launch& l : L.obs) {
      if (l.kind == L_FETCH) {
        if (e->comm) fetch_partner(l.d.xglob);
        continue;
      }
      for (int sh = 0; sh < nsh; ++sh) {
        const ShardView v = view(sh);
        PassDesc d = l.d;
        d.rank_bits = v.rank_bits;
        const double2* src = v.psi;
        const bool reads_partner = l.d.xglob && (l.kind != L_PROD || l.prod_first);
        if (reads_partner) src = e->comm ? scratch : psi + ((uint64_t(sh) ^ (l.d.xglob >> nloc)) << nloc);
        if (reads_partner && emulate) {  // partner shard -> scratch, as fetch_partner does over NCCL
          CK(cudaMemcpyAsync(scratch, src, shard_amps * sizeof(double2), cudaMemcpyDeviceToDevice, s));
          src = scratch;
        }
        if (l.kind == L_PROD) {
          double2* pb = prodbuf + sh * shard_amps;
          double2 scalar = make_double2(0.0, 0.0);
          if (l.prod.last) {  // rank-bit factors: Pauli-basis weights, signs from the source shard's rank bits
            const uint64_t src_rank = v.rank_bits ^ l.d.xglob;
            for (const auto& zw : l.prod_z) {
              const double2 w = __builtin_popcountll(src_rank & zw.first) & 1 ? make_double2(-zw.second.x, -zw.second.y)
                                                                               : zw.second;
              scalar = make_double2(scalar.x + w.x, scalar.y + w.y);
            }
            scalar = cm(l.prod_coeff, scalar);
          }
          launch_prod(d, l.prod, l.grid, l.smem, s, l.prod_first ? src : pb, pb, v.psi, v.lam, scalar, v.part);
          ++launches;
          continue;
        }
        if (l.kind == L_OBS_DIRECT) {
          launch_obs_direct(d, l.grid, s, v.psi, src, v.lam, dterms, v.part);
        } else if (l.jit) {
          const JitObsArgsHead head{v.psi, src, v.lam, v.part, d.part_off, d.rank_bits, d.xglob};
          std::vector<unsigned char> args = jit_obs_args(*l.jit, head, L.terms.data() + d.op_begin);
          launch_generated(l.jit->fn, l.grid, kThreads, l.smem, s, args);
          ++jit_launches;
        } else {
          launch_obs(d, l.grid, l.smem, s, v.psi, src, v.lam, dterms, v.part);
        }
        ++launches;
      }
    }
    CK(cudaEventRecord(e->ev[3], s));
    for (const Launch& l : L.rev) {
      if (l.kind == L_SWAP) {
        swap_pair(l.gbit, l.lpos);
        continue;
      }
      for (int sh = 0; sh < nsh; ++sh) {
        const ShardView v = view(sh);
        PassDesc d = l.d;
        d.rank_bits = v.rank_bits;
        if (l.kind == L_REG)
          launch_reg(l, d, v.psi, v.lam, v.part);
        else
          launch_rev(d, l.grid, l.smem, s, v.psi, v.lam, dops, dcoef, v.part);
        ++launches;
      }
    }
    CK(cudaEventRecord(e->ev[4], s));
    for (int sh = 0; sh < nsh; ++sh) {
      launch_finalize(view(sh).part, dsums, static_cast<int>(cnt), dres + sh * cnt, s);
      ++launches;
    }
    CK(cudaGetLastError());
    // per-shard results -> every rank (NCCL) -> host, summed in shard order (deterministic)
    int nres = nsh;
    const double2* dsrc = dres;
    if (e->comm) {
      double2* dall = static_cast<double2*>(e->gathered.ptr);
      nccl->check(nccl->all_gather(dres, dall, cnt * 2, kNcclFloat64, e->comm, s), "ncclAllGather");
      nres = world;
      dsrc = dall;
    }
    double2* hres = static_cast<double2*>(e->hres.ptr);
    CK(cudaMemcpyAsync(hres, dsrc, cnt * nres * sizeof(double2), cudaMemcpyDeviceToHost, s));
    d2h += cnt * nres * sizeof(double2);
    CK(cudaEventRecord(e->ev[5], s));
    CK(cudaStreamSynchronize(s));
    std::vector<double2> tot(cnt, make_double2(0.0, 0.0));
    for (int r = 0; r < nres; ++r)
      for (int64_t i = 0; i < cnt; ++i) {
        tot[i].x += hres[r * cnt + i].x;
        tot[i].y += hres[r * cnt + i].y;
      }

    // numeric guard: a non-finite partial makes its finalized sum non-finite
    int32_t nonfinite = 0;
    for (int r = 0; r < nres; ++r)
      for (int64_t i = 0; i < cnt; ++i)
        nonfinite += !(std::isfinite(hres[r * cnt + i].x) && std::isfinite(hres[r * cnt + i].y));
    const int A = with_reverse ? p->num_derivs : 0;
    if (energy_out) *energy_out = svg_c128{tot[A].x, tot[A].y};
    if (with_reverse) {
      if (deriv_out)
        for (int d = 0; d < A; ++d) deriv_out[d] = svg_c128{tot[d].x, tot[d].y};
      if (sums_out) {
        for (int q = 0; q < p->num_params; ++q) sums_out[q] = svg_c128{0.0, 0.0};
        // reference order: gates descending, local parameters ascending (gradients.py:158-165)
        std::vector<int> first(p->num_gates + 1, 0);
        for (int i = 0; i < p->num_gates; ++i) first[i + 1] = first[i] + p->gates[i].nderiv;
        for (int i = p->num_gates - 1; i >= 0; --i)
          for (int j = 0; j < p->gates[i].nderiv; ++j) {
            const int d = first[i] + j;
            svg_c128& dst = sums_out[p->derivs[d].param_ref];
            dst.re += tot[d].x;
            dst.im += tot[d].y;
          }
      }
    }
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->ms_total = elapsed(e->ev[0], e->ev[5]);
      stats->ms_forward = elapsed(e->ev[1], e->ev[2]);
      stats->ms_observable = elapsed(e->ev[2], e->ev[3]);
      stats->ms_reverse = elapsed(e->ev[3], e->ev[4]);
      stats->ms_other = stats->ms_total - stats->ms_forward - stats->ms_observable - stats->ms_reverse;
      stats->launches = launches;
      int fp = 0, rp = 0, op = 0;
      for (const Launch& l : L.fwd) fp += l.kind != L_SWAP;
      for (const Launch& l : L.rev) rp += l.kind != L_SWAP;
      for (const Launch& l : L.obs) op += l.kind != L_FETCH;
      stats->fwd_passes = fp;
      stats->obs_passes = op;
      stats->rev_passes = rp;
      stats->tile_qubits = L.k;
      stats->segments = L.reg ? static_cast<int32_t>(L.segs.size()) : 0;
      stats->reg_bits = L.reg ? L.R : 0;
      stats->pass_bytes = L.pass_bytes * nsh;
      stats->h2d_bytes = h2d;
      stats->d2h_bytes = d2h;
      stats->swaps = L.swaps;
      stats->exchange_bytes = L.swap_bytes;
      stats->jit_passes = jit_launches;
      stats->ms_host_lower = std::chrono::duration<double, std::milli>(t_lowered - t_enter).count();
      stats->ms_host_prep = std::chrono::duration<double, std::milli>(t_launch - t_lowered).count();
      stats->nonfinite = nonfinite;
    }
    return SVG_OK;
  } catch (const InvalidArg& ex) {
    return fail(SVG_EINVAL, ex.what());
  } catch (const CudaError& ex) {
    return fail(ex.code == cudaErrorMemoryAllocation ? SVG_ENOMEM : SVG_ECUDA, ex.what());
  } catch (const JitFailure& ex) {
    return fail(SVG_ECUDA, std::string("generated kernels: ") + ex.what());
  } catch (const NcclError& ex) {
    // a failed exchange leaves the peers mid-collective: abort the communicator so
    // no rank blocks on it; the engine cannot run sharded sweeps afterwards
    if (e->comm) {
      const Nccl& nc = Nccl::get();
      if (nc.comm_abort) nc.comm_abort(e->comm);
      e->comm = nullptr;
    }
    return fail(SVG_ENCCL, ex.what());
  } catch (const std::bad_alloc&) {
    return fail(SVG_ENOMEM, "host allocation failed");
  } catch (const std::exception& ex) {
    return fail(SVG_ECUDA, ex.what());
  }
}

}  // namespace

extern "C" {

int svg_abi_version(void) { return SVG_ABI_VERSION; }

const char* svg_last_error(void) { return g_last_error.c_str(); }

int svg_device_count(int* out) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (out) *out = 0;
    return fail(SVG_EUNSUPPORTED, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  if (out) *out = c;
  return SVG_OK;
}

int svg_engine_create(int device, svg_engine** out) {
  if (!out) return fail(SVG_EINVAL, "null out pointer");
  *out = nullptr;
  int count = 0;
  if (svg_device_count(&count) != SVG_OK) return SVG_EUNSUPPORTED;
  if (device < 0 || device >= count) return fail(SVG_EINVAL, "device index out of range");
  svg_engine* e = new (std::nothrow) svg_engine();
  if (!e) return fail(SVG_ENOMEM, "host allocation failed");
  try {
    e->device = device;
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) throw InvalidArg("this build targets sm_100a (B200); found sm_" +
                                          std::to_string(prop.major * 10 + prop.minor));
    e->sms = prop.multiProcessorCount;
    e->max_smem = prop.sharedMemPerBlockOptin;
    e->max_smem_sm = prop.sharedMemPerMultiprocessor;
    CK(prepare_kernels(e->max_smem));
    CK(prepare_reg_kernels(e->max_smem));
    CK(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking));
    e->stream = e->own_stream;
    for (auto& ev : e->ev) CK(cudaEventCreate(&ev));
  } catch (const InvalidArg& ex) {
    delete e;
    return fail(SVG_EUNSUPPORTED, ex.what());
  } catch (const CudaError& ex) {
    delete e;
    return fail(SVG_ECUDA, ex.what());
  }
  *out = e;
  return SVG_OK;
}

static int log2_shards(int shards) {
  if (shards < 1 || (shards & (shards - 1))) return -1;
  return __builtin_ctz(static_cast<unsigned>(shards));
}

int svg_engine_create_virtual(int device, int shards, svg_engine** out) {
  const int g = log2_shards(shards);
  if (g < 0 || g > 6) return fail(SVG_EINVAL, "shards must be a power of two <= 64");
  const int rc = svg_engine_create(device, out);
  if (rc != SVG_OK) return rc;
  (*out)->shard_bits = g;
  (*out)->shards_local = shards;
  return SVG_OK;
}

int svg_nccl_unique_id(uint8_t id_out[128]) {
  if (!id_out) return fail(SVG_EINVAL, "null id buffer");
  try {
    NcclUniqueId id;
    const Nccl& nc = Nccl::get();
    nc.check(nc.get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, sizeof(id.internal));
    return SVG_OK;
  } catch (const std::exception& ex) {
    return fail(SVG_ENCCL, ex.what());
  }
}

int svg_engine_create_sharded(int device, int world, int rank, const uint8_t nccl_id[128], svg_engine** out) {
  const int g = log2_shards(world);
  if (g < 0 || g > 6) return fail(SVG_EINVAL, "world size must be a power of two <= 64");
  if (rank < 0 || rank >= world || !nccl_id) return fail(SVG_EINVAL, "bad rank or null NCCL id");
  const int rc = svg_engine_create(device, out);
  if (rc != SVG_OK) return rc;
  svg_engine* e = *out;
  e->shard_bits = g;
  e->shards_local = 1;
  e->rank = rank;
  {  // world 1 too: a one-rank communicator runs the same all-gather path
    try {
      NcclUniqueId id;
      std::memcpy(id.internal, nccl_id, sizeof(id.internal));
      const Nccl& nc = Nccl::get();
      nc.check(nc.comm_init_rank(&e->comm, world, id, rank), "ncclCommInitRank");
    } catch (const std::exception& ex) {
      svg_engine_destroy(e);
      *out = nullptr;
      return fail(SVG_ENCCL, ex.what());
    }
  }
  return SVG_OK;
}

int svg_engine_destroy(svg_engine* e) {
  if (!e) return SVG_OK;
  cudaSetDevice(e->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  if (e->comm) Nccl::get().comm_destroy(e->comm);
  e->scratch.release();
  e->gathered.release();
  e->prodbuf.release();
  e->psi.release();
  e->lam.release();
  e->partials.release();
  e->blob.release();
  e->results.release();
  e->hblob.release();
  e->hres.release();
  for (auto& ev : e->ev)
    if (ev) cudaEventDestroy(ev);
  if (e->blob_ev) cudaEventDestroy(e->blob_ev);
  for (cudaEvent_t ev : e->chunk_ev)
    if (ev) cudaEventDestroy(ev);
  if (e->enter_ev) cudaEventDestroy(e->enter_ev);
  if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
  if (e->own_stream) cudaStreamDestroy(e->own_stream);
  delete e;
  return SVG_OK;
}

int svg_engine_set_stream(svg_engine* e, void* stream) {
  if (!e) return fail(SVG_EINVAL, "null engine");
  e->stream = stream ? static_cast<cudaStream_t>(stream) : e->own_stream;
  return SVG_OK;
}

int svg_engine_set_option(svg_engine* e, const char* key, int64_t value) {
  if (!e || !key) return fail(SVG_EINVAL, "null argument");
  const std::string k(key);
  if (k == "tile_qubits") {
    if (value < 0 || value > 13) return fail(SVG_EINVAL, "tile_qubits must be in [0, 13]");
    e->opt_tile = value;
  } else if (k == "profile") {
    e->opt_profile = value;
  } else if (k == "reg_bits") {
    if (value != 0 && value != 3 && value != 4) return fail(SVG_EINVAL, k + " must be 0 (auto), 3 or 4");
    e->opt_reg_bits = value;
  } else if (k == "emulate_transport") {
    e->opt_emulate_transport = value != 0;
  } else if (k == "kernel") {
    if (value < 0 || value > 2) return fail(SVG_EINVAL, "kernel must be 0 (auto), 1 (shared-memory tiles) or 2 (register tiles)");
    e->opt_kernel = value;
  } else if (k == "tile_fwd") {
    if (value < -1 || value > 13) return fail(SVG_EINVAL, "tile_fwd must be in [-1, 13]");
    e->opt_tile_fwd = value;
  } else if (k == "checked") {
    e->opt_checked = value != 0;
  } else if (k == "low_qubits") {
    if (value < 3 || value > 5) return fail(SVG_EINVAL, "low_qubits must be in [3, 5]");
    e->opt_low_qubits = value;
  } else if (k == "jit") {
    if (value < 0 || value > 2) return fail(SVG_EINVAL, "jit must be 0 (off), 1 (auto) or 2 (always)");
    e->opt_jit = value;
  } else if (k == "max_gates_per_pass") {
    if (value < 0) return fail(SVG_EINVAL, "max_gates_per_pass must be >= 0");
    e->opt_max_items = value;
  } else {
    return fail(SVG_EINVAL, "unknown option " + k);
  }
  return SVG_OK;
}

int svg_reverse_sweep(svg_engine* e, const svg_problem* p, svg_c128* sums_out, svg_c128* deriv_out,
                      svg_c128* energy_out, svg_stats* stats) {
  return run(e, p, true, sums_out, deriv_out, energy_out, stats);
}

int svg_expectation(svg_engine* e, const svg_problem* p, svg_c128* energy_out, svg_stats* stats) {
  return run(e, p, false, nullptr, nullptr, energy_out, stats);
}

int svg_plan_schedule(const svg_problem* p, int shards, int tile_qubits, int sms, int32_t* order_out,
                      int32_t* step_start_out, int32_t* step_swap_out, uint64_t* qmask_out, int32_t* nsteps_out,
                      int32_t* tile_qubits_out) {
  try {
    validate(p);
    const int g = log2_shards(shards);
    if (g < 0) throw InvalidArg("shards must be a power of two");
    const int n = p->num_qubits, nloc = n - g;
    PlanParams pp;
    pp.n = nloc;
    pp.k = choose_tile_qubits(nloc, tile_qubits, sms > 0 ? sms : 148);
    pp.b = (nloc <= pp.k) ? nloc : std::min(5, pp.k - 2);
    std::vector<GateShape> shapes(p->num_gates);
    for (int i = 0; i < p->num_gates; ++i) shapes[i] = gate_shape(p->gates[i]);
    const std::vector<Step> steps = plan_schedule(shapes, n, g, pp, nullptr);
    int pos = 0;
    for (size_t j = 0; j < steps.size(); ++j) {
      if (step_start_out) step_start_out[j] = pos;
      // swap steps: (gbit << 8 | lpos) + 1; pass steps: 0
      if (step_swap_out) step_swap_out[j] = steps[j].swap ? ((steps[j].gbit << 8) | steps[j].lpos) + 1 : 0;
      if (qmask_out) qmask_out[j] = steps[j].swap ? 0 : steps[j].pass.qmask;
      if (!steps[j].swap)
        for (int gi : steps[j].pass.items) {
          if (order_out) order_out[pos] = gi;
          ++pos;
        }
    }
    if (step_start_out) step_start_out[steps.size()] = pos;
    if (nsteps_out) *nsteps_out = static_cast<int32_t>(steps.size());
    if (tile_qubits_out) *tile_qubits_out = pp.k;
    return SVG_OK;
  } catch (const std::exception& ex) {
    return fail(SVG_EINVAL, ex.what());
  }
}

// Debug / test hook (not in the public header): lower `p` on a device-less
// engine with circuit-specialised kernels forced on, generate and NVRTC-compile
// every distinct pass kernel (nothing is loaded).  opts: tile_qubits, reg_bits,
// reg_bits_fwd, acc_kb (0: engine defaults).  *npasses = register passes covered.
extern "C" int svg_debug_jit_check(const svg_problem* p, const int64_t* opts, int32_t* npasses) {
  try {
    validate(p);
    svg_engine e;
    e.sms = 148;
    e.max_smem = 232448;
    e.opt_jit = 2;
    e.jit_dry_run = true;
    if (opts) {
      e.opt_tile = opts[0];
      e.opt_reg_bits = opts[1];
      e.opt_checked = opts[2];
    }
    (void)lower(&e, p, true);
    (void)cudaGetLastError();
    if (npasses) *npasses = e.jit_dry_count;
    if (e.jit_error != "dry run") return fail(SVG_EINVAL, "generated kernels: " + e.jit_error);
    return SVG_OK;
  } catch (const std::exception& ex) {
    return fail(SVG_EINVAL, ex.what());
  }
}

// Debug / tools (not in the public header): the shape of the plan the engine would
// run with generated kernels (no GPU, nothing compiled).  opts: tile_qubits, reg_bits,
// low_qubits, max_gates_per_pass, pass_windows (0/1), log2(shards).  out[0..7] forward,
// out[8..15] reverse: passes, segments, layout changes, register ops, lane flips,
// max slots, passes with lane-group accumulators.
extern "C" int svg_debug_plan_stats(const svg_problem* p, const int64_t* opts, double* out) {
  try {
    validate(p);
    svg_engine e;
    e.sms = 148;
    e.max_smem = 232448;
    e.max_smem_sm = 233472;
    e.opt_jit = 2;
    e.jit_dry_run = 2;
    e.opt_tile = opts[0];
    e.opt_reg_bits = opts[1];
    if (opts[2]) e.opt_low_qubits = opts[2];
    e.opt_max_items = opts[3];
    e.opt_windows = opts[4];
    e.shard_bits = static_cast<int>(opts[5]);
    (void)lower(&e, p, true);
    (void)cudaGetLastError();
    for (int i = 0; i < 16; ++i) out[i] = e.plan_stats[i];
    return SVG_OK;
  } catch (const std::exception& ex) {
    return fail(SVG_EINVAL, ex.what());
  }
}

// Debug / tests (not in the public header): the free-lane segment plan of one pass.
// flips / touch: tile-local masks of the pass's m gates in order; out_seg[i] = segment
// of gate i, out_pos[i] = its position inside the segment; regmask / lanemask per segment.
extern "C" int svg_debug_segments(const uint32_t* flips, const uint32_t* touch, int m, int k, int regbits, int lowb,
                                  int32_t* out_seg, int32_t* out_pos, uint32_t* regmask, uint32_t* lanemask,
                                  int32_t* nsegs) {
  try {
    const std::vector<uint32_t> f(flips, flips + m), t(touch, touch + m);
    const std::vector<Segment> segs = plan_segments_free(f, t, k, regbits, lowb);
    for (int i = 0; i < m; ++i) out_seg[i] = out_pos[i] = -1;
    for (size_t s = 0; s < segs.size(); ++s) {
      regmask[s] = segs[s].regmask;
      lanemask[s] = segs[s].lanemask;
      for (size_t j = 0; j < segs[s].items.size(); ++j) {
        out_seg[segs[s].items[j]] = static_cast<int32_t>(s);
        out_pos[segs[s].items[j]] = static_cast<int32_t>(j);
      }
    }
    *nsegs = static_cast<int32_t>(segs.size());
    return SVG_OK;
  } catch (const std::exception& ex) {
    return fail(SVG_EINVAL, ex.what());
  }
}

// Debug / profiling (not in the public header): per-phase host milliseconds of
// lower() accumulated on the calling thread since the last reset (out_ms[0..8]).
extern "C" int svg_debug_phase_ms(double* out_ms, int reset) {
  for (int i = 0; i < 9; ++i) out_ms[i] = g_phase_ms[i];
  if (reset)
    for (double& v : g_phase_ms) v = 0.0;
  return SVG_OK;
}

// Debug / profiling (not in the public header): host-only lowering of `p`
// `reps` times on a device-less engine (interpreted kernels, no CUDA calls
// that matter); out_ms[0..7] = accumulated per-phase milliseconds.
extern "C" int svg_debug_lower_timing(const svg_problem* p, int reps, double* out_ms) {
  try {
    validate(p);
    svg_engine e;
    e.sms = 148;
    e.max_smem = 232448;
    e.opt_jit = 0;
    for (double& v : g_phase_ms) v = 0.0;
    for (int r = 0; r < reps; ++r) (void)lower(&e, p, true);
    for (int i = 0; i < 8; ++i) out_ms[i] = g_phase_ms[i];
    (void)cudaGetLastError();
    return SVG_OK;
  } catch (const std::exception& ex) {
    return fail(SVG_EINVAL, ex.what());
  }
}

int svg_plan_inspect(const svg_problem* p, int tile_qubits, int sms, int32_t* order_out,
                     int32_t* pass_start_out, uint64_t* qmask_out, int32_t* npasses_out,
                     int32_t* tile_qubits_out) {
  try {
    validate(p);
    const int n = p->num_qubits;
    PlanParams pp;
    pp.n = n;
    pp.k = choose_tile_qubits(n, tile_qubits, sms > 0 ? sms : 148);
    pp.b = (n <= pp.k) ? n : std::min(5, pp.k - 2);
    std::vector<GateShape> shapes(p->num_gates);
    for (int i = 0; i < p->num_gates; ++i) shapes[i] = gate_shape(p->gates[i]);
    const std::vector<Pass> passes = plan_gate_passes(shapes, pp);
    int pos = 0;
    for (size_t j = 0; j < passes.size(); ++j) {
      if (pass_start_out) pass_start_out[j] = pos;
      if (qmask_out) qmask_out[j] = passes[j].qmask;
      for (int g : passes[j].items) {
        if (order_out) order_out[pos] = g;
        ++pos;
      }
    }
    if (pass_start_out) pass_start_out[passes.size()] = pos;
    if (npasses_out) *npasses_out = static_cast<int32_t>(passes.size());
    if (tile_qubits_out) *tile_qubits_out = pp.k;
    return SVG_OK;
  } catch (const std::exception& ex) {
    return fail(SVG_EINVAL, ex.what());
  }
}

}  // extern "C"
