// Register-tile building blocks shared by the interpreted pass kernel
// (kernels_reg.cu) and the circuit-specialised pass kernels generated at run
// time (jit.cpp, compiled with NVRTC): register layouts, tile load / store /
// transposes, and the per-op register arithmetic.
#pragma once
#include "device.cuh"
#include "tile_ops.cuh"

namespace svgb {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double2 shfl2(double2 v, uint32_t m) {
  return make_double2(__shfl_xor_sync(kFull, v.x, m), __shfl_xor_sync(kFull, v.y, m));
}
// flip the sign of both components when bit `s` (0/1) is set (sign-bit xor, no FP op)
__device__ __forceinline__ double2 sflip(double2 v, uint32_t s) {
  const long long m = static_cast<long long>(s) << 63;
  return make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ m),
                      __longlong_as_double(__double_as_longlong(v.y) ^ m));
}

template <int R>
struct Map {
  uint64_t gw;        // global offset of this warp's warp bits
  uint64_t gbit[R];   // global offset of register bit i
  uint32_t sw;        // tile-local offset of the warp bits
  uint32_t sbit[R];   // tile-local offset of register bit i
};

template <int R>
__device__ __forceinline__ void make_map(Map<R>& m, const SegDesc& sg, const uint8_t* sq, int warp, int wbits) {
  m.gw = 0;
  m.sw = 0;
  for (int i = 0; i < wbits; ++i)
    if ((warp >> i) & 1) {
      m.gw |= 1ull << sq[sg.warppos[i]];
      m.sw |= 1u << sg.warppos[i];
    }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    m.gbit[i] = 1ull << sq[sg.regpos[i]];
    m.sbit[i] = 1u << sg.regpos[i];
  }
}

template <int R>
__device__ __forceinline__ uint64_t goff(const Map<R>& m, int j) {
  uint64_t o = 0;
#pragma unroll
  for (int i = 0; i < R; ++i)
    if ((j >> i) & 1) o |= m.gbit[i];
  return o;
}
template <int R>
__device__ __forceinline__ uint32_t soff(const Map<R>& m, int j) {
  uint32_t o = 0;
#pragma unroll
  for (int i = 0; i < R; ++i)
    if ((j >> i) & 1) o |= m.sbit[i];
  return o;
}

template <int R>
__device__ __forceinline__ void load_g(double2 (&v)[1 << R], const double2* __restrict__ g, uint64_t row,
                                       const Map<R>& m) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) v[j] = g[row + goff(m, j)];  // disjoint bits: + folds into offsets
}
template <int R>
__device__ __forceinline__ void store_g(const double2 (&v)[1 << R], double2* __restrict__ g, uint64_t row,
                                        const Map<R>& m) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) g[row + goff(m, j)] = v[j];
}
template <int R>
__device__ __forceinline__ void to_smem(const double2 (&v)[1 << R], double2* s, uint32_t row, const Map<R>& m) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) s[row + soff(m, j)] = v[j];
}
template <int R>
__device__ __forceinline__ void from_smem(double2 (&v)[1 << R], const double2* s, uint32_t row, const Map<R>& m) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) v[j] = s[row + soff(m, j)];
}

// Per-op, per-thread constants.
struct OpCtx {
  double a, bb;    // CTRL: new = a v + bb (i^BI) p ; otherwise new = v + bb (i^BI) p (bb = t, scaled form)
  uint32_t pneg;   // permutation modes: sign of bb (bb = +-1)
  uint32_t smask;  // register part of the partner sign (runtime patterns only)
  uint32_t cmask;  // register part of the control test
  bool clw_ok;     // lane/warp part of the control test
};

// Register-op patterns: flip shape and how the partner sign depends on the
// register slot j.  Compile-time sign patterns cost nothing (negated FMA
// operands); only the rare multi-bit Z patterns read the runtime smask.
//   P_DIAG            diagonal, sign uniform
//   P_DIAGZ + b       diagonal, sign_j = bit_b(j)               (RZ-type on register bit b)
//   P_LANE            lane flip, sign uniform
//   P_REG + b         flip register bit b, sign uniform         (RX-type)
//   P_REGY + b        flip register bit b, sign_j = !bit_b(j)   (RY-type: Z on the flipped bit)
//   P_GDIAG / P_GLANE / P_GREG + b   runtime smask
template <int R>
struct Pat {
  static constexpr int DIAG = 0, DIAGZ = 1, LANE = 1 + R, REG = 2 + R, REGY = 2 + 2 * R, GDIAG = 2 + 3 * R,
                       GLANE = 3 + 3 * R, GREG = 4 + 3 * R, N = 4 + 4 * R;
};

// One amplitude update with partner p and partner sign (-1)^neg:
//   SC (scaled form, uncontrolled rotations):  v + t (i^BI p)   -- one DFMA per component;
//      the gate's uniform factor a is deferred: the tile holds psi / C, C = product of
//      the a's since the last flush (host-tracked, applied at the segment's flush point,
//      and folded as C^2 into the inner-product coefficients);
//   !SC (controlled / small-a ops):           a v + bb (i^BI p);
//   BI 3/4: pure Pauli (a = 0, |b'| = 1), a signed permutation without arithmetic.
template <int BI, bool SC>
__device__ __forceinline__ double2 upd(const OpCtx& c, double2 v, double2 p, bool neg) {
  if (BI >= 3) {
    const uint32_t s = uint32_t(neg) ^ c.pneg;
    return BI == 3 ? sflip(p, s) : sflip(make_double2(-p.y, p.x), s);
  }
  const double t = neg ? -c.bb : c.bb;
  const double px = BI == 1 ? -p.y : p.x, py = BI == 1 ? p.x : p.y;
  if (SC) return make_double2(fma(t, px, v.x), fma(t, py, v.y));
  return make_double2(fma(c.a, v.x, t * px), fma(c.a, v.y, t * py));
}

// Inner-product terms for one amplitude: partner p with sign (-1)^neg.
// IPK 1: q += Re(conj(lam) sel(s p)), sel = -i (BI) or 1 ; IPK 3: z += conj(lam) s p, z2 += conj(lam) v.
template <int IPK, int BI>
__device__ __forceinline__ void ip_term(double2 lam, double2 p, double2 v, bool neg, double& q, double2& z,
                                        double2& z2) {
  const double lx = neg ? -lam.x : lam.x, ly = neg ? -lam.y : lam.y;  // sign folded into lambda (free negation)
  if (IPK == 1) {
    if (BI == 1)
      q = fma(lx, p.y, fma(-ly, p.x, q));
    else
      q = fma(lx, p.x, fma(ly, p.y, q));
  } else if (IPK == 3) {
    z.x = fma(lx, p.x, fma(ly, p.y, z.x));
    z.y = fma(lx, p.y, fma(-ly, p.x, z.y));
    z2.x = fma(lam.x, v.x, fma(lam.y, v.y, z2.x));
    z2.y = fma(lam.x, v.y, fma(-lam.y, v.x, z2.y));
  }
}

// Sign of the partner of register slot j for pattern P (compile-time unless runtime pattern).
template <int R, int P>
__device__ __forceinline__ bool psign(const OpCtx& c, int j) {
  using PT = Pat<R>;
  if constexpr (P >= PT::DIAGZ && P < PT::LANE) return (j >> (P - PT::DIAGZ)) & 1;
  else if constexpr (P >= PT::REGY && P < PT::GDIAG) return !((j >> (P - PT::REGY)) & 1);
  else if constexpr (P >= PT::GDIAG) return (c.smask >> j) & 1u;
  else return false;
}

// One op on the register tile v (and, DUAL, the same op on lambda l).  For
// IPK != 0 the inner product uses lambda and phi before the update (phi_{i+1}).
// BI 2 (IPK 3 ops): b' real or imaginary at run time (c.bi).
template <int R, int P, int IPK, int BI, bool CTRL, bool DUAL>
__device__ __forceinline__ void reg_op(double2 (&v)[1 << R], double2 (&l)[1 << R], const OpCtx& c, uint32_t xl,
                                       double (&q)[4], double2& z, double2& z2) {
  using PT = Pat<R>;
  constexpr int NR = 1 << R;
  constexpr bool SC = !CTRL;
  constexpr bool LANEF = (P == PT::LANE || P == PT::GLANE);
  constexpr int XB = (P >= PT::REG && P < PT::GDIAG) ? (P - PT::REG) % R : (P >= PT::GREG ? P - PT::GREG : -1);
  constexpr int XR = XB >= 0 ? (1 << XB) : 0;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if (XR != 0 && (j & XR)) continue;  // register pairs handled at the low member
    const int jp = j ^ XR;
    const bool sj = psign<R, P>(c, j);
    const bool okj = !CTRL || (c.clw_ok && ((c.cmask >> j) & 1u));
    double2 pj = v[jp];  // partner of slot j (slot jp of the partner lane)
    double2 lpj = DUAL ? l[jp] : pj;
    if (LANEF) {
      pj = shfl2(pj, xl);
      if (DUAL) lpj = shfl2(lpj, xl);
    }
    if (IPK != 0 && okj) ip_term<IPK, BI>(l[j], pj, v[j], sj, q[j & 3], z, z2);
    if (XR == 0) {
      if (!CTRL || okj) {
        v[j] = upd<BI, SC>(c, v[j], pj, sj);
        if (DUAL) l[j] = upd<BI, SC>(c, l[j], lpj, sj);
      }
    } else {
      const bool sp = psign<R, P>(c, jp);
      if (IPK != 0 && okj) ip_term<IPK, BI>(l[jp], v[j], v[jp], sp, q[jp & 3], z, z2);
      if (!CTRL || okj) {
        const double2 vj = v[j], lj = l[j];
        v[j] = upd<BI, SC>(c, vj, pj, sj);
        v[jp] = upd<BI, SC>(c, v[jp], vj, sp);
        if (DUAL) {
          l[j] = upd<BI, SC>(c, lj, lpj, sj);
          l[jp] = upd<BI, SC>(c, l[jp], lj, sp);
        }
      }
    }
  }
}

// Where a reverse op's inner product goes.
struct IpSink {
  double* tacc;   // lane-group accumulators [nslots][nthr >> shift] (or null)
  double2* wacc;  // per-warp accumulators [nwarps][nslots]
  int nthr, nslots, warp, lane;
  int shift;      // lanes 2^shift apart are combined (butterfly) before the shared accumulate
};

__device__ __forceinline__ double warp_sum1(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <int R>
__device__ __forceinline__ void scale_tile(double2 (&v)[1 << R], double s) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) v[j] = make_double2(v[j].x * s, v[j].y * s);
}

// One real inner-product contribution of this thread into `slot`.
__device__ __forceinline__ void sink_real(const IpSink& sink, uint32_t slot, double qk) {
  if (sink.tacc) {
    double qa = qk;
    for (int o = 1; o < (1 << sink.shift); o <<= 1) qa += __shfl_xor_sync(kFull, qa, o);
    if ((sink.lane & ((1 << sink.shift) - 1)) == 0)
      sink.tacc[slot * (sink.nthr >> sink.shift) + (threadIdx.x >> sink.shift)] += qa;
  } else {
    const double w = warp_sum1(qk);
    if (sink.lane == 0) sink.wacc[sink.warp * sink.nslots + slot].x += w;
  }
}

// Kernel-local variant id (computed on the host, see engine.cu emit_rop):
//   id = pattern + Pat<R>::N * (ctrl + 2 * mode)
//   forward kernels (NB 1), kFwdModes: 0/1 rotation (BI 0/1), 2/3 signed permutation (BI 0/1)
//   reverse kernels (NB 2), kRevModes: 0/1 rotation + single-component inner product (BI 0/1),
//     2 rotation + complex inner product (IPK 3), 3/4 signed permutation of phi and lambda
// ctrl = 1 selects the unscaled form with control predicates (also used, with an
// all-pass mask, for rotations whose a is too small to defer).
constexpr int kFwdModes = 4, kRevModes = 5;
// RET: a single-component inner product is returned instead of accumulated
// (the generated kernels add it to an accumulator they loaded before the op).
template <int R, int NB, int V, bool RET = false>
__device__ __forceinline__ double op_body(double2 (&v)[1 << R], double2 (&l)[1 << R], const OpCtx& c, uint32_t xl,
                                          uint32_t slw, bool rbi, uint32_t slot, double kr, double2 ka, double2 kb,
                                          const IpSink& sink) {
  constexpr int NP = Pat<R>::N;
  constexpr int P = V % NP;
  constexpr bool CTRL = (V / NP) % 2;
  constexpr int mode = V / NP / 2;
  constexpr bool DUAL = NB == 2;
  constexpr int IPK = !DUAL ? 0 : (mode <= 1 ? 1 : (mode == 2 ? 3 : 0));
  constexpr int BI = !DUAL ? (mode <= 1 ? mode : 3 + (mode - 2)) : (mode <= 1 ? mode : (mode == 2 ? 2 : 3 + (mode - 3)));
  double q[4] = {0.0, 0.0, 0.0, 0.0};  // independent accumulation chains (8 measured 1 % slower)
  double2 z = make_double2(0.0, 0.0), z2 = make_double2(0.0, 0.0);
  if constexpr (BI == 2) {  // IPK 3: b' real or imaginary chosen at run time
    if (rbi)
      reg_op<R, P, 3, 1, CTRL, DUAL>(v, l, c, xl, q, z, z2);
    else
      reg_op<R, P, 3, 0, CTRL, DUAL>(v, l, c, xl, q, z, z2);
  } else {
    reg_op<R, P, IPK, BI, CTRL, DUAL>(v, l, c, xl, q, z, z2);
  }
  if constexpr (IPK == 1) {  // per-thread accumulator: no per-op warp reduction
    const double qs = (q[0] + q[1]) + (q[2] + q[3]);
    if constexpr (RET) return kr * (slw ? -qs : qs);
    sink_real(sink, slot, kr * (slw ? -qs : qs));
  } else if constexpr (IPK == 3) {
    if (slw) z = make_double2(-z.x, -z.y);
    z = warp_sum(z);
    z2 = warp_sum(z2);
    const double2 contrib = cfma(kb, z, cmul(ka, z2));
    if (sink.lane == 0) {
      double2& acc = sink.wacc[sink.warp * sink.nslots + slot];
      acc = make_double2(acc.x + contrib.x, acc.y + contrib.y);
    }
  }
  return 0.0;
}


// Per-CTA slot sums -> partials[s * gridDim.x + blockIdx.x]: one warp per slot,
// lanes stride over the per-warp and lane-group accumulators, then a butterfly
// (fixed order: deterministic).
__device__ __forceinline__ void flush_partials(const double2* wacc, const double* tacc, int nslots, int nwarps,
                                               int nacc, double2* out, int warp, int lane) {
  for (int s = warp; s < nslots; s += nwarps) {
    double x = 0.0, y = 0.0;
    for (int w = lane; w < nwarps; w += 32) {
      x += wacc[w * nslots + s].x;
      y += wacc[w * nslots + s].y;
    }
    if (tacc)
      for (int t = lane; t < nacc; t += 32) x += tacc[s * nacc + t];
    x = warp_sum1(x);
    y = warp_sum1(y);
    if (lane == 0) out[static_cast<long long>(s) * gridDim.x + blockIdx.x] = make_double2(x, y);
  }
}

// ---- asynchronous tile staging (cp.async, 16 B per copy, L1 bypass) ----
// Each thread stages its own 2^R amplitudes of the NEXT tile into a private
// slice of shared memory ([j][thread] layout: conflict-free 16-byte rows) while
// it computes the current tile; cp.async.wait_all then makes them visible to
// the same thread -- no block barrier.
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
template <int R>
__device__ __forceinline__ void stage_g(double2* stg, const double2* __restrict__ g, uint64_t row, const Map<R>& m,
                                        int tid, int nthr) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) cp_async16(stg + j * nthr + tid, g + row + goff(m, j));
}
template <int R>
__device__ __forceinline__ void unstage(double2 (&v)[1 << R], const double2* stg, int tid, int nthr) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) v[j] = stg[j * nthr + tid];
}

// ---- checked mode (engine option "checked"; generated kernels only) ----
// Shared-memory reads poison what they read with a NaN, so a read that comes
// before its write in a later phase (a missing barrier or cp.async wait, a
// wrong swizzle or staging slot) returns NaN and fails the parity check;
// global tile indices are bounds-checked (trap).
__device__ __forceinline__ double2 poison2() {
  return make_double2(__longlong_as_double(0x7ff8dead0000beefll), __longlong_as_double(0x7ff8dead0000beefll));
}
#define SVGB_CHECK(cond) \
  do {                   \
    if (!(cond)) __trap(); \
  } while (0)
template <int R>
__device__ __forceinline__ void unstage_poison(double2 (&v)[1 << R], double2* stg, int tid, int nthr) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) {
    v[j] = stg[j * nthr + tid];
    stg[j * nthr + tid] = poison2();
  }
}
// every global amplitude of a thread's 2^R slots lies below `limit`
template <int R>
__device__ __forceinline__ void check_rows(uint64_t row, const Map<R>& m, uint64_t limit) {
  SVGB_CHECK(row + goff(m, (1 << R) - 1) < limit);
}

// One register op with its structure as template arguments (jit.cpp): the same
// steps as the interpreted kernel's op loop, with every mask a literal.
template <int R, int NB, int V, uint32_t XL, uint32_t ZLW, uint32_t CLW, uint32_t SMASK, uint32_t CMASK,
          uint64_t ZO, uint64_t CO, bool RBI, uint32_t SLOT, bool RET = false, int PSIGN = -1>
__device__ __forceinline__ double jit_op(double2 (&v)[1 << R], double2 (&l)[1 << R], uint64_t sbase, uint32_t tbase,
                                         double ca, double cbb, double kr, double2 ka, double2 kb, const IpSink& sink) {
  if (CO != 0 && (sbase & CO) != CO) return 0.0;
  uint32_t slw = 0;
  if (ZLW != 0) slw ^= uint32_t(__popc((tbase ^ XL) & ZLW));
  if (ZO != 0) slw ^= uint32_t(__popcll(sbase & ZO));
  slw &= 1u;
  OpCtx c;
  c.a = ca;
  c.bb = slw ? -cbb : cbb;
  c.smask = SMASK;
  c.cmask = CMASK;
  c.clw_ok = (tbase & CLW) == CLW;
  // signed permutations (fixed Paulis): the sign is structural and, without
  // lane / warp / off-tile Z factors, a literal (PSIGN 0 / 1) -- no sign flips
  c.pneg = PSIGN >= 0 ? uint32_t(PSIGN) : uint32_t(c.bb < 0.0);
  return op_body<R, NB, V, RET>(v, l, c, XL, slw, RBI, SLOT, kr, ka, kb, sink);
}

}  // namespace svgb
