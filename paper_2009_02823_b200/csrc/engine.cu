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
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/svgrad_b200.h"
#include "device.cuh"
#include "kernels.h"
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

enum LaunchKind { L_SMEM_FWD, L_SMEM_REV, L_OBS, L_OBS_DIRECT, L_REG };

struct Launch {
  PassDesc d;
  int grid = 0;
  size_t smem = 0;
  int kind = L_SMEM_FWD;
  int nb = 1;       // L_REG: buffers in the pass (1 forward, 2 reverse)
  int threads = kThreads;
  int R = 3;           // L_REG: register bits
  bool tiles = false;  // L_REG: stages the tile through shared memory
};

// Everything a sweep needs on the host side, built from one svg_problem.
struct Lowered {
  int n = 0, k = 0, b = 0;
  bool reg = false;  // register-tile kernels in use
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
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int64_t opt_tile = 0, opt_profile = 0, opt_max_items = 0, opt_kernel = 0, opt_reg_bits = 4, opt_reg_bits_fwd = 4, opt_prefetch = 0;
  DeviceBuf psi, lam, partials, blob, results;
  HostBuf hblob, hres;
  cudaEvent_t ev[6] = {};
};

namespace {

void validate(const svg_problem* p) {
  if (!p) throw InvalidArg("null problem");
  const int n = p->num_qubits;
  if (n < 1 || n > SVG_MAX_QUBITS) throw InvalidArg("num_qubits out of range");
  if (p->num_gates < 0 || p->num_derivs < 0 || p->num_terms < 1 || p->num_params < 0)
    throw InvalidArg("negative table size or empty observable");
  if ((p->num_gates && !p->gates) || (p->num_derivs && !p->derivs) || !p->terms)
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

SegDesc make_seg(int kind, uint32_t regmask, int k, int R, SegLocal* sl) {
  sl->R = R;
  SegDesc sd;
  std::memset(&sd, 0, sizeof(sd));
  sd.kind = kind;
  int r = 0, w = 0;
  for (int pos = 0; pos < k; ++pos) {
    if (pos < 5) {
      sl->bit[pos] = static_cast<uint8_t>(pos);
    } else if ((regmask >> pos) & 1) {
      sd.regpos[r] = static_cast<uint8_t>(pos);
      sl->bit[pos] = static_cast<uint8_t>(5 + r++);
    } else {
      sd.warppos[w] = static_cast<uint8_t>(pos);
      sl->bit[pos] = static_cast<uint8_t>(5 + R + w++);
    }
  }
  return sd;
}

// One register op for gate g: operator coefficients `c` (a, b of a I + b P),
// optionally fused with the post-gate generator `kpost` into `slot`.
void emit_rop(Lowered& L, const TileMap& tm, const SegLocal& sl, const svg_gate& g, uint32_t kind,
              const svg_c128* c, const svg_c128* kpost, uint32_t slot, bool real_sums) {
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
  uint32_t mode = perm ? 2 + (bi ? 1 : 0) : (bi ? 1 : 0);
  if (kind == ROP_REV) {
    if (op.flags & RF_IP3)
      mode = 6;
    else if (op.flags & RF_IP1)
      mode = 4 + (bi ? 1 : 0);
    else if (perm)
      mode = 7 + (bi ? 1 : 0);
    else
      throw std::logic_error("parameter-free non-permutation Pauli op reached the register path");
  }
  op.variant = pattern + NP * ((cloc != 0) + 2 * mode);
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

Lowered lower(const svg_engine* e, const svg_problem* p, bool with_reverse) {
  Lowered L;
  const int n = p->num_qubits;
  const bool real_sums = (p->flags & SVG_FLAG_REAL_SUMS) != 0;
  L.n = n;
  L.k = choose_tile_qubits(n, static_cast<int>(e->opt_tile), e->sms);
  L.b = (n <= L.k) ? n : std::min(5, L.k - 2);
  const int RB = static_cast<int>(e->opt_reg_bits);      // reverse passes
  const int RF = static_cast<int>(e->opt_reg_bits_fwd);  // forward passes
  L.R = RB;
  auto fits = [&](int R) { return L.k - 5 - R >= 0 && (32 << (L.k - 5 - R)) <= reg_max_threads(R); };
  L.reg = e->opt_kernel != 1 && L.b >= 5 && fits(RB) && fits(RF);
  if (e->opt_kernel == 2 && !L.reg) throw InvalidArg("register-tile kernels need 5 + reg_bits .. 13 tile qubits");
  PlanParams pp;
  pp.n = n;
  pp.k = L.k;
  pp.b = L.b;
  if (e->opt_max_items > 0) pp.max_items = static_cast<int>(e->opt_max_items);
  const int64_t S = int64_t(16) << n;

  std::vector<GateShape> shapes(p->num_gates);
  for (int i = 0; i < p->num_gates; ++i) shapes[i] = gate_shape(p->gates[i]);
  const std::vector<Pass> gpasses = plan_gate_passes(shapes, pp);

  std::vector<int> first_deriv(p->num_gates + 1, 0);
  for (int i = 0; i < p->num_gates; ++i) first_deriv[i + 1] = first_deriv[i] + p->gates[i].nderiv;
  std::vector<Gen> gens(p->num_derivs);
  for (int d = 0; d < p->num_derivs; ++d) gens[d] = make_gen(p->gates[p->derivs[d].gate], p->derivs[d]);

  // segments per pass (register path)
  std::vector<std::vector<Segment>> psegs(gpasses.size()), psegs_f(gpasses.size());
  if (L.reg) {
    for (size_t pi = 0; pi < gpasses.size(); ++pi) {
      const Pass& ps = gpasses[pi];
      const TileMap tm = tile_map(ps.qmask);
      std::vector<uint32_t> flips(ps.items.size()), touch(ps.items.size());
      std::vector<char> dense(ps.items.size());
      for (size_t j = 0; j < ps.items.size(); ++j) {
        const svg_gate& g = p->gates[ps.items[j]];
        flips[j] = tm.local(shapes[ps.items[j]].flip);
        touch[j] = tm.local(shapes[ps.items[j]].touch);
        dense[j] = !reg_capable(g, flips[j]);
      }
      psegs[pi] = plan_segments(flips, touch, dense, L.k, RB);
      psegs_f[pi] = RF == RB ? psegs[pi] : plan_segments(flips, touch, dense, L.k, RF);
    }
  }
  auto reg_launch = [&](const Pass& ps, int nb) {
    Launch l;
    l.d = make_desc(n, L.k, ps.qmask);
    l.kind = L_REG;
    l.nb = nb;
    l.R = nb == 1 ? RF : RB;
    l.threads = 32 << (L.k - 5 - l.R);
    l.d.seg_begin = static_cast<int>(L.segs.size());
    l.d.op_begin = static_cast<int>(L.rops.size());  // this pass's register ops (staged in smem)
    return l;
  };
  // default register layout for shared-memory segments: lowest non-lane positions
  auto default_regs = [](int R) { return ((1u << (5 + R)) - 1u) & ~31u; };

  // forward passes
  for (size_t pi = 0; pi < gpasses.size(); ++pi) {
    const Pass& ps = gpasses[pi];
    const TileMap tm = tile_map(ps.qmask);
    if (!L.reg) {
      Launch l;
      l.d = make_desc(n, L.k, ps.qmask);
      l.kind = L_SMEM_FWD;
      l.d.op_begin = static_cast<int>(L.ops.size());
      for (int gi : ps.items) emit_op(L, tm, p->gates[gi], OP_APPLY_PAULI, 0, p->gates[gi].fwd, 0);
      l.d.op_end = static_cast<int>(L.ops.size());
      L.fwd.push_back(l);
    } else {
      Launch l = reg_launch(ps, 1);
      uint32_t prev = ~0u;
      for (const Segment& sg : psegs_f[pi]) {
        SegLocal sl;
        SegDesc sd = make_seg(sg.reg ? SEG_REG : SEG_SMEM, sg.reg ? sg.regmask : default_regs(RF), L.k, RF, &sl);
        sd.same_map = sg.reg && sg.regmask == prev;
        prev = sg.reg ? sg.regmask : ~0u;
        if (sg.reg) {
          sd.op_begin = static_cast<int>(L.rops.size());
          for (int it : sg.items) {
            const svg_gate& g = p->gates[ps.items[it]];
            emit_rop(L, tm, sl, g, ROP_FWD, g.fwd, nullptr, 0, real_sums);
          }
          sd.op_end = static_cast<int>(L.rops.size());
        } else {
          sd.op_begin = static_cast<int>(L.ops.size());
          for (int it : sg.items) emit_op(L, tm, p->gates[ps.items[it]], OP_APPLY_PAULI, 0, p->gates[ps.items[it]].fwd, 0);
          sd.op_end = static_cast<int>(L.ops.size());
          l.tiles = true;
        }
        L.segs.push_back(sd);
      }
      l.d.seg_end = static_cast<int>(L.segs.size());
      l.d.op_end = static_cast<int>(L.rops.size());
      if (psegs_f[pi].size() > 1) l.tiles = true;
      L.fwd.push_back(l);
    }
    L.pass_bytes += 2 * S;
  }

  // observable passes (terms grouped by flip mask into tiles)
  std::vector<uint64_t> flips(p->num_terms);
  for (int t = 0; t < p->num_terms; ++t) flips[t] = p->terms[t].x_mask;
  std::vector<int> direct;
  std::vector<Pass> tpasses = plan_term_passes(flips, pp, &direct);
  if (!direct.empty()) {  // wide flip masks: one untiled gather pass (qmask 0)
    Pass ps;
    ps.items = direct;
    tpasses.push_back(ps);
  }
  int64_t part = 0;
  const int64_t energy_off = 0;
  for (size_t j = 0; j < tpasses.size(); ++j) {
    const Pass& ps = tpasses[j];
    const TileMap tm = tile_map(ps.qmask);
    Launch l;
    l.d = make_desc(n, L.k, ps.qmask);
    l.d.op_begin = static_cast<int>(L.terms.size());
    l.d.untiled = ps.qmask == 0;
    l.kind = l.d.untiled ? L_OBS_DIRECT : L_OBS;
    for (int ti : ps.items) {
      const svg_pauli_term& src = p->terms[ti];
      DevTerm dt;
      dt.c = cm(d2(src.coeff), ipow(src.n_y));
      if (l.d.untiled) {  // full masks: x split over (xl, zl), z in zo
        dt.xl = static_cast<uint32_t>(src.x_mask);
        dt.zl = static_cast<uint32_t>(src.x_mask >> 32);
        dt.zo = src.z_mask;
      } else {
        dt.xl = tm.local(src.x_mask);
        dt.zl = tm.local(src.z_mask);
        dt.zo = src.z_mask & ~tm.qmask;
      }
      L.terms.push_back(dt);
    }
    l.d.op_end = static_cast<int>(L.terms.size());
    l.d.accumulate = j > 0;
    L.obs.push_back(l);
    L.pass_bytes += (j > 0 ? 3 : 2) * S;
  }

  // reverse passes: forward passes backwards, gates backwards inside
  std::vector<std::pair<int, int>> deriv_slot(p->num_derivs, {-1, -1});  // (rev pass, slot)
  auto smem_reverse_ops = [&](const TileMap& tm, int gi, uint32_t& slot) {
    const svg_gate& g = p->gates[gi];
    emit_op(L, tm, g, OP_APPLY_PAULI, 0, g.rewind, 0);
    for (int j = 0; j < g.nderiv; ++j) {
      const int d = first_deriv[gi] + j;
      deriv_slot[d] = {static_cast<int>(L.rev.size()), static_cast<int>(slot)};
      emit_op(L, tm, g, OP_IP_PAULI, 0, gens[d].pre, slot++);
    }
    if (gi > 0) emit_op(L, tm, g, OP_APPLY_PAULI, 1, g.adjoint, 0);
  };
  if (with_reverse) {
    for (int pi = static_cast<int>(gpasses.size()) - 1; pi >= 0; --pi) {
      const Pass& ps = gpasses[pi];
      const TileMap tm = tile_map(ps.qmask);
      uint32_t slot = 0;
      if (!L.reg) {
        Launch l;
        l.d = make_desc(n, L.k, ps.qmask);
        l.kind = L_SMEM_REV;
        l.d.op_begin = static_cast<int>(L.ops.size());
        for (auto it = ps.items.rbegin(); it != ps.items.rend(); ++it) smem_reverse_ops(tm, *it, slot);
        l.d.op_end = static_cast<int>(L.ops.size());
        l.d.nslots = static_cast<int>(slot);
        L.rev.push_back(l);
      } else {
        Launch l = reg_launch(ps, 2);
        const std::vector<Segment>& sgs = psegs[pi];
        uint32_t prev = ~0u;
        for (auto st = sgs.rbegin(); st != sgs.rend(); ++st) {
          const Segment& sg = *st;
          SegLocal sl;
          SegDesc sd = make_seg(sg.reg ? SEG_REG : SEG_SMEM, sg.reg ? sg.regmask : default_regs(RB), L.k, RB, &sl);
          sd.same_map = sg.reg && sg.regmask == prev;
          prev = sg.reg ? sg.regmask : ~0u;
          if (sg.reg) {
            sd.op_begin = static_cast<int>(L.rops.size());
            for (auto it = sg.items.rbegin(); it != sg.items.rend(); ++it) {
              const int gi = ps.items[*it];
              const svg_gate& g = p->gates[gi];
              const svg_c128* kpost = nullptr;
              if (g.nderiv == 1) {
                const int d = first_deriv[gi];
                deriv_slot[d] = {static_cast<int>(L.rev.size()), static_cast<int>(slot)};
                kpost = gens[d].post;
              }
              // one op rewinds phi AND lambda (rewind == adjoint for register-capable gates);
              // the reference skips lambda's update at i = 0, whose value is never read again
              emit_rop(L, tm, sl, g, ROP_REV, g.rewind, kpost, kpost ? slot++ : 0, real_sums);
            }
            sd.op_end = static_cast<int>(L.rops.size());
          } else {
            sd.op_begin = static_cast<int>(L.ops.size());
            for (auto it = sg.items.rbegin(); it != sg.items.rend(); ++it) smem_reverse_ops(tm, ps.items[*it], slot);
            sd.op_end = static_cast<int>(L.ops.size());
            l.tiles = true;
          }
          L.segs.push_back(sd);
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

  // grids, shared memory, partial offsets
  const int64_t ntiles = int64_t(1) << (n - L.k);
  auto clamp_grid = [&](int per_sm) {
    const int64_t slots = int64_t(e->sms) * per_sm;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, slots)));
  };
  auto size_launch = [&](Launch& l) {
    switch (l.kind) {
      case L_SMEM_FWD:
        l.smem = fwd_smem(L.k, l.d.b);
        l.grid = clamp_grid(occupancy(0, l.smem));
        break;
      case L_SMEM_REV:
        l.smem = rev_smem(L.k, l.d.b, l.d.nslots);
        l.grid = clamp_grid(occupancy(2, l.smem));
        break;
      case L_REG:
        // per-thread inner-product accumulators when they fit a modest budget
        l.d.thread_acc = l.nb == 2 && size_t(l.d.nslots) * l.threads * sizeof(double) <= (48u << 10);
        l.d.prefetch = e->opt_prefetch != 0;
        l.smem = reg_smem(L.k, l.d.b, l.nb, l.threads / 32, l.d.nslots, l.d.op_end - l.d.op_begin, l.tiles,
                          l.d.thread_acc != 0, l.d.prefetch != 0);
        l.grid = clamp_grid(reg_occupancy(l.nb, l.R, l.threads, l.smem));
        break;
      case L_OBS:
        l.smem = obs_smem(L.k, l.d.b);
        l.grid = clamp_grid(occupancy(1, l.smem));
        break;
      default:
        l.smem = 0;
        l.grid = std::max(1, static_cast<int>(std::min<int64_t>(int64_t(e->sms) * 8, int64_t(1) << std::max(0, n - 8))));
    }
    if (l.smem > e->max_smem) throw InvalidArg("pass needs more shared memory than the device offers");
  };
  for (Launch& l : L.fwd) size_launch(l);
  for (Launch& l : L.obs) {
    size_launch(l);
    l.d.part_off = part;
    part += l.grid;
  }
  const int64_t energy_count = part - energy_off;
  for (Launch& l : L.rev) {
    size_launch(l);
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

int run(svg_engine* e, const svg_problem* p, bool with_reverse, svg_c128* sums_out,
        svg_c128* deriv_out, svg_c128* energy_out, svg_stats* stats) {
  if (!e) return fail(SVG_EINVAL, "null engine");
  try {
    validate(p);
    CK(cudaSetDevice(e->device));
    const Lowered L = lower(e, p, with_reverse);
    const int n = L.n;
    const size_t amps = size_t(1) << n;
    cudaStream_t s = e->stream;

    e->psi.reserve(amps * sizeof(double2));
    e->lam.reserve(amps * sizeof(double2));
    e->partials.reserve(std::max<int64_t>(1, L.partial_count) * sizeof(double2));
    const Blob bl = layout(L);
    e->blob.reserve(bl.total);
    e->hblob.reserve(bl.total);
    e->results.reserve(L.sums.size() * sizeof(double2));
    e->hres.reserve(L.sums.size() * sizeof(double2));

    char* hb = static_cast<char*>(e->hblob.ptr);
    char* db = static_cast<char*>(e->blob.ptr);
    // the pinned staging buffer may still feed a previous call's copy
    CK(cudaStreamSynchronize(s));
    std::memcpy(hb + bl.ops, L.ops.data(), L.ops.size() * sizeof(DevOp));
    std::memcpy(hb + bl.coef, L.coef.data(), L.coef.size() * sizeof(double2));
    std::memcpy(hb + bl.terms, L.terms.data(), L.terms.size() * sizeof(DevTerm));
    std::memcpy(hb + bl.sums, L.sums.data(), L.sums.size() * sizeof(SumSpec));
    std::memcpy(hb + bl.rops, L.rops.data(), L.rops.size() * sizeof(RegOp));
    std::memcpy(hb + bl.segs, L.segs.data(), L.segs.size() * sizeof(SegDesc));

    double2* psi = static_cast<double2*>(e->psi.ptr);
    double2* lam = static_cast<double2*>(e->lam.ptr);
    double2* part = static_cast<double2*>(e->partials.ptr);
    const DevOp* dops = reinterpret_cast<const DevOp*>(db + bl.ops);
    const double2* dcoef = reinterpret_cast<const double2*>(db + bl.coef);
    const DevTerm* dterms = reinterpret_cast<const DevTerm*>(db + bl.terms);
    const SumSpec* dsums = reinterpret_cast<const SumSpec*>(db + bl.sums);
    const RegOp* drops = reinterpret_cast<const RegOp*>(db + bl.rops);
    const SegDesc* dsegs = reinterpret_cast<const SegDesc*>(db + bl.segs);
    double2* dres = static_cast<double2*>(e->results.ptr);

    int64_t launches = 0, h2d = bl.total, d2h = L.sums.size() * sizeof(double2);
    CK(cudaEventRecord(e->ev[0], s));
    CK(cudaMemcpyAsync(db, hb, bl.total, cudaMemcpyHostToDevice, s));
    if (p->input_amps) {
      CK(cudaMemcpyAsync(psi, p->input_amps, amps * sizeof(double2), cudaMemcpyHostToDevice, s));
      h2d += amps * sizeof(double2);
    } else {
      CK(cudaMemsetAsync(psi, 0, amps * sizeof(double2), s));
      launch_set_basis(psi, static_cast<uint64_t>(p->input_basis), s);
      launches += 1;
    }
    CK(cudaEventRecord(e->ev[1], s));
    for (const Launch& l : L.fwd) {
      if (l.kind == L_REG)
        launch_pass_reg(1, l.R, l.d, l.grid, l.threads, l.smem, s, psi, nullptr, dsegs, drops, dops, dcoef, part);
      else
        launch_fwd(l.d, l.grid, l.smem, s, psi, dops, dcoef);
    }
    CK(cudaEventRecord(e->ev[2], s));
    for (const Launch& l : L.obs) {
      if (l.d.untiled)
        launch_obs_direct(l.d, l.grid, s, psi, lam, dterms, part);
      else
        launch_obs(l.d, l.grid, l.smem, s, psi, lam, dterms, part);
    }
    CK(cudaEventRecord(e->ev[3], s));
    for (const Launch& l : L.rev) {
      if (l.kind == L_REG)
        launch_pass_reg(2, l.R, l.d, l.grid, l.threads, l.smem, s, psi, lam, dsegs, drops, dops, dcoef, part);
      else
        launch_rev(l.d, l.grid, l.smem, s, psi, lam, dops, dcoef, part);
    }
    CK(cudaEventRecord(e->ev[4], s));
    launch_finalize(part, dsums, static_cast<int>(L.sums.size()), dres, s);
    CK(cudaGetLastError());
    launches += L.fwd.size() + L.obs.size() + L.rev.size() + 1;
    double2* hres = static_cast<double2*>(e->hres.ptr);
    CK(cudaMemcpyAsync(hres, dres, L.sums.size() * sizeof(double2), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(e->ev[5], s));
    CK(cudaStreamSynchronize(s));

    const int A = with_reverse ? p->num_derivs : 0;
    if (energy_out) *energy_out = svg_c128{hres[A].x, hres[A].y};
    if (with_reverse) {
      if (deriv_out)
        for (int d = 0; d < A; ++d) deriv_out[d] = svg_c128{hres[d].x, hres[d].y};
      if (sums_out) {
        for (int q = 0; q < p->num_params; ++q) sums_out[q] = svg_c128{0.0, 0.0};
        // reference order: gates descending, local parameters ascending (gradients.py:158-165)
        std::vector<int> first(p->num_gates + 1, 0);
        for (int i = 0; i < p->num_gates; ++i) first[i + 1] = first[i] + p->gates[i].nderiv;
        for (int i = p->num_gates - 1; i >= 0; --i)
          for (int j = 0; j < p->gates[i].nderiv; ++j) {
            const int d = first[i] + j;
            svg_c128& dst = sums_out[p->derivs[d].param_ref];
            dst.re += hres[d].x;
            dst.im += hres[d].y;
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
      stats->fwd_passes = static_cast<int32_t>(L.fwd.size());
      stats->obs_passes = static_cast<int32_t>(L.obs.size());
      stats->rev_passes = static_cast<int32_t>(L.rev.size());
      stats->tile_qubits = L.k;
      stats->segments = L.reg ? static_cast<int32_t>(L.segs.size()) : 0;
      stats->reg_bits = L.reg ? L.R : 0;
      stats->pass_bytes = L.pass_bytes;
      stats->h2d_bytes = h2d;
      stats->d2h_bytes = d2h;
    }
    return SVG_OK;
  } catch (const InvalidArg& ex) {
    return fail(SVG_EINVAL, ex.what());
  } catch (const CudaError& ex) {
    return fail(ex.code == cudaErrorMemoryAllocation ? SVG_ENOMEM : SVG_ECUDA, ex.what());
  } catch (const std::bad_alloc&) {
    return fail(SVG_ENOMEM, "host allocation failed");
  } catch (const std::exception& ex) {
    return fail(SVG_EINVAL, ex.what());
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

int svg_engine_destroy(svg_engine* e) {
  if (!e) return SVG_OK;
  cudaSetDevice(e->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  e->psi.release();
  e->lam.release();
  e->partials.release();
  e->blob.release();
  e->results.release();
  e->hblob.release();
  e->hres.release();
  for (auto& ev : e->ev)
    if (ev) cudaEventDestroy(ev);
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
  } else if (k == "reg_bits" || k == "reg_bits_fwd") {
    if (value == 0) value = 4;
    if (value != 3 && value != 4) return fail(SVG_EINVAL, k + " must be 3 or 4");
    (k == "reg_bits" ? e->opt_reg_bits : e->opt_reg_bits_fwd) = value;
  } else if (k == "prefetch") {
    e->opt_prefetch = value != 0;
  } else if (k == "kernel") {
    if (value < 0 || value > 2) return fail(SVG_EINVAL, "kernel must be 0 (auto), 1 (shared-memory tiles) or 2 (register tiles)");
    e->opt_kernel = value;
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
