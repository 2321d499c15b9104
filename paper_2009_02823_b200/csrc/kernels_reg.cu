// Register-tile pass kernel for sm_100a: the hot K1/K3 path.
//
// One CTA processes 2^k-amplitude tiles (k = 5 lane + R register + w warp
// bits, see device.cuh).  Per tile:
//   global -> registers (512-byte coalesced rows: lanes are qubits 0..4)
//   for each segment: run its Pauli-form gates entirely in registers --
//       register-bit flips are register pairs (one code path per flipped
//       register bit), lane-bit flips are warp shuffles, Z factors and
//       controls are sign / predicate bits precomputed on the host per
//       register slot; the reverse step fuses  slot += <lam|K'|phi>  and
//       phi <- R phi  on the same partner values, then  lam <- U^dag lam
//       (svgrad/gradients.py:158-168; generator form of svgrad/circuit.py:316-334;
//       the probe mu never exists);
//   between segments: transpose through shared memory (one barrier);
//   dense-matrix gates (Phase, H, callables, 2-bit register flips) run on
//   the shared-memory tile with the generic tile ops;
//   registers -> global.
// A pass with one register segment touches shared memory only for the
// per-warp inner-product accumulators.
#include <cuda_runtime.h>

#include "device.cuh"
#include "kernels.h"
#include "tile_ops.cuh"

namespace svgb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kRegThreads = 256;  // launch bound: k = 11 tiles with R = 3 (8 warps)

__device__ __forceinline__ double2 shfl2(double2 v, uint32_t m) {
  return make_double2(__shfl_xor_sync(kFull, v.x, m), __shfl_xor_sync(kFull, v.y, m));
}
// flip the sign of both components when bit `s` (0/1) is set (sign-bit xor, no FP op)
__device__ __forceinline__ double2 sflip(double2 v, uint32_t s) {
  const long long m = static_cast<long long>(s) << 63;
  return make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ m),
                      __longlong_as_double(__double_as_longlong(v.y) ^ m));
}

// ---- async bulk copies (TMA engine, cp.async.bulk) completing on an mbarrier ----
__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Warp 0 streams tile `base` (rows of 2^b contiguous amplitudes) into the stage buffers.
template <int NB>
__device__ __forceinline__ void prefetch_tile(const PassDesc& d, const uint64_t* rows, uint64_t base,
                                              const double2* b0, const double2* b1, double2* st0, double2* st1,
                                              uint64_t* bar) {
  // one elected thread issues every row (the bulk-copy operands live in uniform registers)
  if ((threadIdx.x & 31) != 0) return;
  const int nrows = 1 << (d.k - d.b);
  const uint32_t row_bytes = uint32_t(sizeof(double2)) << d.b;
  fence_async_smem();  // order earlier generic-proxy smem accesses before the async writes
  mbar_expect_tx(bar, uint32_t(NB) * uint32_t(nrows) * row_bytes);
  for (int r = 0; r < nrows; ++r) {
    const uint64_t g = base | rows[r];
    bulk_g2s(st0 + (size_t(r) << d.b), b0 + g, row_bytes, bar);
    if (NB == 2) bulk_g2s(st1 + (size_t(r) << d.b), b1 + g, row_bytes, bar);
  }
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
  for (int j = 0; j < (1 << R); ++j) v[j] = g[row | goff(m, j)];
}
template <int R>
__device__ __forceinline__ void store_g(const double2 (&v)[1 << R], double2* __restrict__ g, uint64_t row,
                                        const Map<R>& m) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) g[row | goff(m, j)] = v[j];
}
template <int R>
__device__ __forceinline__ void to_smem(const double2 (&v)[1 << R], double2* s, uint32_t row, const Map<R>& m) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) s[row | soff(m, j)] = v[j];
}
template <int R>
__device__ __forceinline__ void from_smem(double2 (&v)[1 << R], const double2* s, uint32_t row, const Map<R>& m) {
#pragma unroll
  for (int j = 0; j < (1 << R); ++j) v[j] = s[row | soff(m, j)];
}

// Per-op, per-thread constants.
struct OpCtx {
  double a, bb;    // new = a v + bb * (i^BI) * p   (bb carries the uniform part of the partner sign)
  double2 bc;      // generic complex b' (reverse mode 6)
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

// v <- a v + (-1)^neg bb (i^BI p)      (in-place friendly: the DFMA overwrites v)
template <int BI>
__device__ __forceinline__ double2 upd(const OpCtx& c, double2 v, double2 p, bool neg) {
  if (BI >= 3) {  // pure Pauli (a = 0, |b'| = 1): a signed permutation, no arithmetic
    const uint32_t s = uint32_t(neg) ^ c.pneg;
    return BI == 3 ? sflip(p, s) : sflip(make_double2(-p.y, p.x), s);
  }
  double tx, ty;
  if (BI == 1) {
    tx = -c.bb * p.y;
    ty = c.bb * p.x;
  } else if (BI == 0) {
    tx = c.bb * p.x;
    ty = c.bb * p.y;
  } else {
    tx = fma(c.bc.x, p.x, -c.bc.y * p.y);
    ty = fma(c.bc.x, p.y, c.bc.y * p.x);
  }
  if (neg) {
    tx = -tx;
    ty = -ty;
  }
  return make_double2(fma(c.a, v.x, tx), fma(c.a, v.y, ty));
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
template <int R, int P, int IPK, int BI, bool CTRL, bool DUAL>
__device__ __forceinline__ void reg_op(double2 (&v)[1 << R], double2 (&l)[1 << R], const OpCtx& c, uint32_t xl,
                                       double& q0, double& q1, double2& z, double2& z2) {
  using PT = Pat<R>;
  constexpr int NR = 1 << R;
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
    if (IPK != 0 && okj) ip_term<IPK, BI>(l[j], pj, v[j], sj, (j & 1) ? q1 : q0, z, z2);
    if (XR == 0) {
      if (!CTRL || okj) {
        v[j] = upd<BI>(c, v[j], pj, sj);
        if (DUAL) l[j] = upd<BI>(c, l[j], lpj, sj);
      }
    } else {
      const bool sp = psign<R, P>(c, jp);
      if (IPK != 0 && okj) ip_term<IPK, BI>(l[jp], v[j], v[jp], sp, q1, z, z2);
      if (!CTRL || okj) {
        const double2 vj = v[j], lj = l[j];
        v[j] = upd<BI>(c, vj, pj, sj);
        v[jp] = upd<BI>(c, v[jp], vj, sp);
        if (DUAL) {
          l[j] = upd<BI>(c, lj, lpj, sj);
          l[jp] = upd<BI>(c, l[jp], lj, sp);
        }
      }
    }
  }
}

// Flat variant id (computed on the host, see engine.cu emit_rop):
//   id = pattern + Pat<R>::N * (ctrl + 2 * mode)
//   mode: forward 0/1 (BI 0/1), 2/3 (signed permutation, BI 0/1: pure Pauli X/Y/Z, CX...);
//         reverse 4/5 (IPK 1, BI 0/1), 6 (IPK 3, generic complex coefficients),
//         7/8 (signed permutation on phi and lambda, BI 0/1)
constexpr int kModes = 9;
template <int R, int NB, int V>
__device__ __forceinline__ void run_variant(double2 (&v)[1 << R], double2 (&l)[1 << R], const OpCtx& c, uint32_t xl,
                                            double& q0, double& q1, double2& z, double2& z2) {
  constexpr int NP = Pat<R>::N;
  if constexpr (V < NP * 2 * kModes) {
    constexpr int P = V % NP;
    constexpr bool CTRL = (V / NP) % 2;
    constexpr int mode = V / NP / 2;
    constexpr bool DUAL = mode >= 4;
    constexpr int IPK = mode == 6 ? 3 : ((mode == 4 || mode == 5) ? 1 : 0);
    constexpr int BI = mode == 6 ? 2 : (mode == 2 || mode == 7) ? 3 : (mode == 3 || mode == 8) ? 4 : (mode & 1);
    // forward kernels only hold forward modes, reverse kernels only reverse modes (code size)
    if constexpr ((NB == 2) == DUAL) reg_op<R, P, IPK, BI, CTRL, DUAL>(v, l, c, xl, q0, q1, z, z2);
  }
}

#define SVGB_V1(N) \
  case (N):        \
    run_variant<R, NB, (N)>(v, l, c, xl, q0, q1, z, z2); \
    break;
#define SVGB_V4(N) SVGB_V1(N) SVGB_V1(N + 1) SVGB_V1(N + 2) SVGB_V1(N + 3)
#define SVGB_V16(N) SVGB_V4(N) SVGB_V4(N + 4) SVGB_V4(N + 8) SVGB_V4(N + 12)
#define SVGB_V64(N) SVGB_V16(N) SVGB_V16(N + 16) SVGB_V16(N + 32) SVGB_V16(N + 48)

template <int R, int NB>
__device__ __forceinline__ void dispatch(uint32_t id, double2 (&v)[1 << R], double2 (&l)[1 << R], const OpCtx& c,
                                         uint32_t xl, double& q0, double& q1, double2& z, double2& z2) {
  static_assert(Pat<R>::N * 2 * kModes <= 384, "extend the dispatch table");
  switch (id) {
    SVGB_V64(0)
    SVGB_V64(64)
    SVGB_V64(128)
    SVGB_V64(192)
    SVGB_V64(256)
    SVGB_V64(320)
    default:
      break;
  }
}
#undef SVGB_V64
#undef SVGB_V16
#undef SVGB_V4
#undef SVGB_V1

__device__ __forceinline__ double warp_sum1(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

}  // namespace

template <int R, int NB>
__global__ void __launch_bounds__(R == 3 ? kRegThreads : kRegThreads / 2, R == 3 ? 2 : (NB == 2 ? 2 : 4)) k_pass_reg(double2* __restrict__ b0, double2* __restrict__ b1,
                                                             const PassDesc d, const SegDesc* __restrict__ segs,
                                                             const RegOp* __restrict__ rops,
                                                             const DevOp* __restrict__ ops,
                                                             const double2* __restrict__ coef,
                                                             double2* __restrict__ partials) {
  constexpr int NR = 1 << R;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint8_t sq[kMaxQubits];
  const int nthr = blockDim.x;
  const int nwarps = nthr >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wbits = d.k - 5 - R;
  double2* wacc = reinterpret_cast<double2*>(smem_raw);  // [nwarps][nslots]
  RegOp* sops = reinterpret_cast<RegOp*>(wacc + nwarps * d.nslots);  // this pass's register ops
  const int nops = d.op_end - d.op_begin;
  double* tacc = d.thread_acc ? reinterpret_cast<double*>(sops + nops) : nullptr;  // [nslots][nthr]
  double2* st0 = reinterpret_cast<double2*>(sops + nops) + (d.thread_acc ? (d.nslots * nthr + 1) / 2 : 0);
  double2* st1 = st0 + (1u << d.k);  // shared tiles (multi-segment passes)
  for (int i = threadIdx.x; i < nwarps * d.nslots; i += nthr) wacc[i] = make_double2(0.0, 0.0);
  if (tacc)
    for (int i = threadIdx.x; i < d.nslots * nthr; i += nthr) tacc[i] = 0.0;
  {
    const uint4* src = reinterpret_cast<const uint4*>(rops + d.op_begin);
    uint4* dst = reinterpret_cast<uint4*>(sops);
    for (int i = threadIdx.x; i < nops * int(sizeof(RegOp) / 16); i += nthr) dst[i] = src[i];
  }
  if (threadIdx.x < kMaxQubits) sq[threadIdx.x] = d.q[threadIdx.x];
  __shared__ uint64_t mbar;
  uint64_t* rows = reinterpret_cast<uint64_t*>(st1 + (NB == 2 ? (1u << d.k) : 0));  // [2^(k-b)] row offsets
  if (d.prefetch) {
    for (int r = threadIdx.x; r < (1 << (d.k - d.b)); r += nthr) {
      uint64_t off = 0;
      for (int j = d.b; j < d.k; ++j)
        if ((r >> (j - d.b)) & 1) off |= 1ull << d.q[j];
      rows[r] = off;
    }
    if (threadIdx.x == 0) mbar_init(&mbar);
  }
  __syncthreads();
  if (d.prefetch && warp == 0) prefetch_tile<NB>(d, rows, pdep64(blockIdx.x, d.rest), b0, b1, st0, st1, &mbar);
  uint32_t phase = 0;

  const uint32_t tbase = uint32_t(lane) | (uint32_t(warp) << (5 + R));
  double2 v[NR], l[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) l[j] = make_double2(0.0, 0.0);
  const uint64_t ntiles = 1ull << (d.n - d.k);
  for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
    const uint64_t base = pdep64(T, d.rest);
    const uint64_t sbase = base | d.rank_bits;  // physical index bits for Z-signs / controls
    const uint64_t next = T + gridDim.x;
    Map<R> m;
    make_map<R>(m, segs[d.seg_begin], sq, warp, wbits);
    if (d.prefetch) {  // this tile was streamed into the stage buffers by the async copy engine
      mbar_wait(&mbar, phase);
      phase ^= 1u;
      from_smem<R>(v, st0, lane | m.sw, m);
      if (NB == 2) from_smem<R>(l, st1, lane | m.sw, m);
    } else {
      load_g<R>(v, b0, base | lane | m.gw, m);
      if (NB == 2) load_g<R>(l, b1, base | lane | m.gw, m);
    }
    bool in_smem = false;
    for (int s = d.seg_begin; s < d.seg_end; ++s) {
      const SegDesc sg = segs[s];
      const bool last = s + 1 == d.seg_end;
      if (sg.kind == SEG_REG) {
        if (s != d.seg_begin && (in_smem || !sg.same_map)) {
          if (!in_smem) {
            __syncthreads();
            to_smem<R>(v, st0, lane | m.sw, m);
            if (NB == 2) to_smem<R>(l, st1, lane | m.sw, m);
          }
          __syncthreads();
          make_map<R>(m, sg, sq, warp, wbits);
          from_smem<R>(v, st0, lane | m.sw, m);
          if (NB == 2) from_smem<R>(l, st1, lane | m.sw, m);
          in_smem = false;
        }
        if (last && d.prefetch && next < ntiles) {  // stage buffers free: stream the next tile
          __syncthreads();
          if (warp == 0) prefetch_tile<NB>(d, rows, pdep64(next, d.rest), b0, b1, st0, st1, &mbar);
        }
        for (int o = sg.op_begin - d.op_begin; o < sg.op_end - d.op_begin; ++o) {
          const RegOp& op = sops[o];
          if ((sbase & op.co) != op.co) continue;
          const uint32_t slw = uint32_t(__popc((tbase ^ op.xl) & op.zlw) ^ __popcll(sbase & op.zo)) & 1u;
          OpCtx c;
          c.a = op.a;
          c.bb = slw ? -op.bb : op.bb;  // uniform part of the partner sign
          c.bc = (op.flags & RF_BI) ? make_double2(0.0, c.bb) : make_double2(c.bb, 0.0);
          c.smask = op.smask;
          c.cmask = op.cmask;
          c.clw_ok = (tbase & op.clw) == op.clw;
          c.pneg = c.bb < 0.0;
          double q0 = 0.0, q1 = 0.0;
          double2 z = make_double2(0.0, 0.0), z2 = make_double2(0.0, 0.0);
          dispatch<R, NB>(op.variant, v, l, c, op.xl, q0, q1, z, z2);
          if constexpr (NB == 2) {
            if (op.flags & RF_IP1) {  // per-thread accumulator: no per-op warp reduction
              const double q = op.kr * (slw ? -(q0 + q1) : q0 + q1);
              if (tacc) {
                tacc[op.slot * nthr + threadIdx.x] += q;
              } else {
                const double w = warp_sum1(q);
                if (lane == 0) wacc[warp * d.nslots + op.slot].x += w;
              }
            } else if (op.flags & RF_IP3) {
              if (slw) z = make_double2(-z.x, -z.y);
              z = warp_sum(z);
              z2 = warp_sum(z2);
              const double2 contrib = cfma(op.kb, z, cmul(op.ka, z2));
              if (lane == 0) {
                double2& acc = wacc[warp * d.nslots + op.slot];
                acc = make_double2(acc.x + contrib.x, acc.y + contrib.y);
              }
            }
          }
        }
      } else {  // SEG_SMEM: generic dense-matrix ops on the shared-memory tile
        if (!in_smem) {
          __syncthreads();
          to_smem<R>(v, st0, lane | m.sw, m);
          if (NB == 2) to_smem<R>(l, st1, lane | m.sw, m);
          __syncthreads();
          in_smem = true;
        }
        for (int o = sg.op_begin; o < sg.op_end; ++o) {
          const DevOp op = ops[o];
          if ((sbase & op.co) != op.co) continue;
          if (op.kind <= OP_APPLY_MAT2) {
            tile_apply(op.buf ? st1 : st0, d.k, op, coef + op.coef, sbase);
          } else {
            const double2 val = warp_sum(tile_ip(st0, st1, d.k, op, coef + op.coef, sbase));
            if (lane == 0) {
              double2& acc = wacc[warp * d.nslots + op.slot];
              acc = make_double2(acc.x + val.x, acc.y + val.y);
            }
          }
          __syncthreads();
        }
        if (last && d.prefetch) {
          from_smem<R>(v, st0, lane | m.sw, m);
          if (NB == 2) from_smem<R>(l, st1, lane | m.sw, m);
          in_smem = false;
          __syncthreads();
          if (warp == 0 && next < ntiles) prefetch_tile<NB>(d, rows, pdep64(next, d.rest), b0, b1, st0, st1, &mbar);
        }
      }
    }
    if (in_smem) {
      from_smem<R>(v, st0, lane | m.sw, m);
      if (NB == 2) from_smem<R>(l, st1, lane | m.sw, m);
    }
    store_g<R>(v, b0, base | lane | m.gw, m);
    if (NB == 2) store_g<R>(l, b1, base | lane | m.gw, m);
  }
  if (d.nslots == 0) return;
  __syncthreads();
  for (int s = threadIdx.x; s < d.nslots; s += nthr) {
    double2 acc = make_double2(0.0, 0.0);
    for (int w = 0; w < nwarps; ++w) {
      const double2 val = wacc[w * d.nslots + s];
      acc = make_double2(acc.x + val.x, acc.y + val.y);
    }
    if (tacc)
      for (int t = 0; t < nthr; ++t) acc.x += tacc[s * nthr + t];
    partials[d.part_off + static_cast<int64_t>(s) * gridDim.x + blockIdx.x] = acc;
  }
}

#define SVGB_INST(R, NB)                                                                                   \
  template __global__ void k_pass_reg<R, NB>(double2*, double2*, const PassDesc, const SegDesc*, const RegOp*, \
                                             const DevOp*, const double2*, double2*);
SVGB_INST(3, 1)
SVGB_INST(3, 2)
SVGB_INST(4, 1)
SVGB_INST(4, 2)
#undef SVGB_INST

namespace {
const void* reg_kernel(int nb, int R) {
  if (R == 4) return nb == 1 ? reinterpret_cast<const void*>(k_pass_reg<4, 1>) : reinterpret_cast<const void*>(k_pass_reg<4, 2>);
  return nb == 1 ? reinterpret_cast<const void*>(k_pass_reg<3, 1>) : reinterpret_cast<const void*>(k_pass_reg<3, 2>);
}

cudaError_t allow_dynamic_smem(const void* fn, size_t max_smem) {
  cudaFuncAttributes attr;
  cudaError_t e = cudaFuncGetAttributes(&attr, fn);
  if (e != cudaSuccess) return e;
  const size_t room = max_smem > attr.sharedSizeBytes ? max_smem - attr.sharedSizeBytes : 0;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(room));
}
}  // namespace

size_t reg_smem(int k, int b, int nb, int nwarps, int nslots, int nops, bool tiles, bool thread_acc, bool prefetch) {
  const size_t tacc = thread_acc ? sizeof(double2) * ((size_t(nslots) * nwarps * 32 + 1) / 2) : 0;
  const size_t rows = prefetch ? sizeof(uint64_t) << (k - b) : 0;
  return sizeof(double2) * (size_t(nwarps) * nslots + ((tiles || prefetch) ? (size_t(nb) << k) : 0)) +
         sizeof(RegOp) * nops + tacc + rows;
}

int reg_max_threads(int R) { return R == 3 ? kRegThreads : kRegThreads / 2; }

cudaError_t prepare_reg_kernels(size_t max_smem) {
  for (int R = 3; R <= 4; ++R)
    for (int nb = 1; nb <= 2; ++nb) {
      const cudaError_t e = allow_dynamic_smem(reg_kernel(nb, R), max_smem);
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}

int reg_occupancy(int nb, int R, int threads, size_t smem) {
  int blocks = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, reg_kernel(nb, R), threads, smem);
  return blocks < 1 ? 1 : blocks;
}

void launch_pass_reg(int nb, int R, const PassDesc& d, int grid, int threads, size_t smem, cudaStream_t s, double2* b0,
                     double2* b1, const SegDesc* segs, const RegOp* rops, const DevOp* ops, const double2* coef,
                     double2* partials) {
  if (R == 4) {
    if (nb == 1)
      k_pass_reg<4, 1><<<grid, threads, smem, s>>>(b0, b1, d, segs, rops, ops, coef, partials);
    else
      k_pass_reg<4, 2><<<grid, threads, smem, s>>>(b0, b1, d, segs, rops, ops, coef, partials);
  } else {
    if (nb == 1)
      k_pass_reg<3, 1><<<grid, threads, smem, s>>>(b0, b1, d, segs, rops, ops, coef, partials);
    else
      k_pass_reg<3, 2><<<grid, threads, smem, s>>>(b0, b1, d, segs, rops, ops, coef, partials);
  }
}

}  // namespace svgb
