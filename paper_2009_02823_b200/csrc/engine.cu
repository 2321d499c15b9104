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

struct Launch {
  PassDesc d;
  int grid;
  size_t smem;
};

// Everything a sweep needs on the host side, built from one svg_problem.
struct Lowered {
  int n = 0, k = 0, b = 0;
  std::vector<DevOp> ops;
  std::vector<double2> coef;
  std::vector<DevTerm> terms;
  std::vector<SumSpec> sums;  // [num_derivs] derivative terms, then [1] energy
  std::vector<Launch> fwd, obs, rev;
  int64_t partial_count = 0;
  int64_t pass_bytes = 0;
};

}  // namespace

struct svg_engine {
  int device = 0;
  int sms = 148;
  size_t max_smem = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int64_t opt_tile = 0, opt_profile = 0, opt_max_items = 0;
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

Lowered lower(const svg_engine* e, const svg_problem* p, bool with_reverse) {
  Lowered L;
  const int n = p->num_qubits;
  L.n = n;
  L.k = choose_tile_qubits(n, static_cast<int>(e->opt_tile), e->sms);
  L.b = (n <= L.k) ? n : std::min(5, L.k - 2);
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

  // forward passes
  for (const Pass& ps : gpasses) {
    const TileMap tm = tile_map(ps.qmask);
    Launch l{make_desc(n, L.k, ps.qmask), 0, 0};
    l.d.op_begin = static_cast<int>(L.ops.size());
    for (int gi : ps.items) emit_op(L, tm, p->gates[gi], OP_APPLY_PAULI, 0, p->gates[gi].fwd, 0);
    l.d.op_end = static_cast<int>(L.ops.size());
    L.fwd.push_back(l);
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
    Launch l{make_desc(n, L.k, ps.qmask), 0, 0};
    l.d.op_begin = static_cast<int>(L.terms.size());
    l.d.untiled = ps.qmask == 0;
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
  if (with_reverse) {
    for (int pi = static_cast<int>(gpasses.size()) - 1; pi >= 0; --pi) {
      const Pass& ps = gpasses[pi];
      const TileMap tm = tile_map(ps.qmask);
      Launch l{make_desc(n, L.k, ps.qmask), 0, 0};
      l.d.op_begin = static_cast<int>(L.ops.size());
      uint32_t slot = 0;
      for (auto it = ps.items.rbegin(); it != ps.items.rend(); ++it) {
        const int gi = *it;
        const svg_gate& g = p->gates[gi];
        emit_op(L, tm, g, OP_APPLY_PAULI, 0, g.rewind, 0);
        for (int j = 0; j < g.nderiv; ++j) {
          const int d = first_deriv[gi] + j;
          deriv_slot[d] = {static_cast<int>(L.rev.size()), static_cast<int>(slot)};
          emit_op(L, tm, g, OP_IP_PAULI, 0, p->derivs[d].k, slot++);
        }
        if (gi > 0) emit_op(L, tm, g, OP_APPLY_PAULI, 1, g.adjoint, 0);
      }
      l.d.op_end = static_cast<int>(L.ops.size());
      l.d.nslots = static_cast<int>(slot);
      L.rev.push_back(l);
      L.pass_bytes += 4 * S;
    }
  }

  // grids, shared memory, partial offsets
  const int64_t ntiles = int64_t(1) << (n - L.k);
  auto grid_for = [&](int which, size_t smem) {
    const int64_t slots = int64_t(e->sms) * occupancy(which, smem);
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, slots)));
  };
  for (Launch& l : L.fwd) {
    l.smem = fwd_smem(L.k, l.d.b);
    l.grid = grid_for(0, l.smem);
  }
  for (Launch& l : L.obs) {
    l.smem = l.d.untiled ? 0 : obs_smem(L.k, l.d.b);
    l.grid = l.d.untiled ? std::max(1, std::min<int>(e->sms * 8, static_cast<int>(std::min<int64_t>(
                               int64_t(1) << std::max(0, n - 8), 1 << 30))))
                         : grid_for(1, l.smem);
    l.d.part_off = part;
    part += l.grid;
  }
  const int64_t energy_count = part - energy_off;
  for (Launch& l : L.rev) {
    l.smem = rev_smem(L.k, l.d.b, l.d.nslots);
    if (l.smem > e->max_smem) throw InvalidArg("pass needs more shared memory than the device offers");
    l.grid = grid_for(2, l.smem);
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
  size_t ops, coef, terms, sums, total;
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

    double2* psi = static_cast<double2*>(e->psi.ptr);
    double2* lam = static_cast<double2*>(e->lam.ptr);
    double2* part = static_cast<double2*>(e->partials.ptr);
    const DevOp* dops = reinterpret_cast<const DevOp*>(db + bl.ops);
    const double2* dcoef = reinterpret_cast<const double2*>(db + bl.coef);
    const DevTerm* dterms = reinterpret_cast<const DevTerm*>(db + bl.terms);
    const SumSpec* dsums = reinterpret_cast<const SumSpec*>(db + bl.sums);
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
    for (const Launch& l : L.fwd) launch_fwd(l.d, l.grid, l.smem, s, psi, dops, dcoef);
    CK(cudaEventRecord(e->ev[2], s));
    for (const Launch& l : L.obs) {
      if (l.d.untiled)
        launch_obs_direct(l.d, l.grid, s, psi, lam, dterms, part);
      else
        launch_obs(l.d, l.grid, l.smem, s, psi, lam, dterms, part);
    }
    CK(cudaEventRecord(e->ev[3], s));
    for (const Launch& l : L.rev) launch_rev(l.d, l.grid, l.smem, s, psi, lam, dops, dcoef, part);
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
