// Register-tile pass kernel (v2) for sm_100a: the hot K1/K3 path.
//
// One CTA processes 2^k-amplitude tiles (k = 5 lane + R register + w warp
// bits, see device.cuh).  Per tile:
//   global -> registers (512-byte coalesced rows: lanes are qubits 0..4)
//   for each segment: run its Pauli-form gates entirely in registers --
//       register-bit flips are register permutations, lane-bit flips are
//       warp shuffles, diagonal factors and controls are index predicates;
//       the reverse step fuses  slot += <lam|K'|phi>,  phi <- R phi  on the
//       same partner values, then  lam <- U^dag lam  (svgrad/gradients.py:158-168,
//       generator form of svgrad/circuit.py:316-334; mu never exists);
//   between segments: transpose through shared memory (one barrier);
//   dense-matrix gates (rare: Phase, H, callables) run on the shared-memory
//   tile with the generic tile ops;
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

__device__ __forceinline__ double2 shfl2(double2 v, uint32_t m) {
  return make_double2(__shfl_xor_sync(kFull, v.x, m), __shfl_xor_sync(kFull, v.y, m));
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

// new = a v + (+-b') p ; ROT: a real, b' real (BI: imaginary -> use i*p and b'.y)
template <bool ROT>
__device__ __forceinline__ double2 combine(double2 a, double2 b, bool bi, double2 v, double2 p, int s) {
  if (ROT) {
    double bb = bi ? b.y : b.x;
    if (s) bb = -bb;
    const double px = bi ? -p.y : p.x, py = bi ? p.x : p.y;
    return make_double2(fma(a.x, v.x, bb * px), fma(a.x, v.y, bb * py));
  }
  return cfma(cneg_if(b, s), p, cmul(a, v));
}

// IPK: 0 none, 1 Re(z) only, 2 Im(z) only, 3 full complex z and z2
template <int IPK>
__device__ __forceinline__ void accumulate(double2& z, double2& z2, double2 lam, double2 p, double2 v, int s) {
  if (IPK == 0) return;
  const double px = s ? -p.x : p.x, py = s ? -p.y : p.y;
  if (IPK == 1 || IPK == 3) z.x = fma(lam.x, px, fma(lam.y, py, z.x));
  if (IPK == 2 || IPK == 3) z.y = fma(lam.x, py, fma(-lam.y, px, z.y));
  if (IPK == 3) z2 = cjfma(lam, v, z2);
}

// One Pauli-form operator on register tile `v` (optionally fused with the
// generator inner product against `l`).  XR: register part of the flip mask.
template <int R, int XR, bool ROT, int IPK>
__device__ __forceinline__ void pauli_step(double2 (&v)[1 << R], const double2 (&l)[1 << R], const RegOp& op,
                                           uint32_t tbase, int sb, double2& z, double2& z2) {
  constexpr int NR = 1 << R;
  constexpr int LOW = XR & -XR;
  const uint32_t xl = op.x & 31u;
  const bool bi = (op.flags & RF_BI) != 0;
  const double2 a = op.a, b = op.b;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if (XR != 0 && (j & LOW)) continue;  // handled with its pair's low member
    const int jp = j ^ XR;
    const uint32_t tj = tbase | (uint32_t(j) << 5);
    double2 pj = v[jp];
    double2 pjp = v[j];
    if (xl) {
      pj = shfl2(pj, xl);
      if (XR != 0) pjp = shfl2(pjp, xl);
    }
    const int sj = par32((tj ^ op.x) & op.z) ^ sb;
    const bool okj = (tj & op.c) == op.c;
    if (okj) accumulate<IPK>(z, z2, l[j], pj, v[j], sj);
    const double2 nj = okj ? combine<ROT>(a, b, bi, v[j], pj, sj) : v[j];
    if (XR != 0) {
      const uint32_t tp = tbase | (uint32_t(jp) << 5);
      const int sp = par32((tp ^ op.x) & op.z) ^ sb;
      if (okj) accumulate<IPK>(z, z2, l[jp], pjp, v[jp], sp);
      v[jp] = okj ? combine<ROT>(a, b, bi, v[jp], pjp, sp) : v[jp];
    }
    v[j] = nj;
  }
}

template <int R, bool ROT, int IPK>
__device__ __forceinline__ void pauli_dispatch(double2 (&v)[1 << R], const double2 (&l)[1 << R], const RegOp& op,
                                               uint32_t tbase, int sb, double2& z, double2& z2) {
  const uint32_t xr = (op.x >> 5) & ((1u << R) - 1u);
  switch (xr) {
#define SVGB_XR(N)                                                        \
  case N:                                                                 \
    if constexpr (N < (1 << R)) pauli_step<R, N, ROT, IPK>(v, l, op, tbase, sb, z, z2); \
    break;
    SVGB_XR(0) SVGB_XR(1) SVGB_XR(2) SVGB_XR(3) SVGB_XR(4) SVGB_XR(5) SVGB_XR(6) SVGB_XR(7)
    SVGB_XR(8) SVGB_XR(9) SVGB_XR(10) SVGB_XR(11) SVGB_XR(12) SVGB_XR(13) SVGB_XR(14) SVGB_XR(15)
#undef SVGB_XR
    default:
      break;
  }
}

template <int R, int IPK>
__device__ __forceinline__ void pauli_op(double2 (&v)[1 << R], const double2 (&l)[1 << R], const RegOp& op,
                                         uint32_t tbase, int sb, double2& z, double2& z2) {
  if (op.flags & RF_ROT)
    pauli_dispatch<R, true, IPK>(v, l, op, tbase, sb, z, z2);
  else
    pauli_dispatch<R, false, IPK>(v, l, op, tbase, sb, z, z2);
}

}  // namespace

template <int R, int NB>
__global__ void __launch_bounds__(256, 1) k_pass_reg(double2* __restrict__ b0, double2* __restrict__ b1,
                                                  const PassDesc d, const SegDesc* __restrict__ segs,
                                                  const RegOp* __restrict__ rops, const DevOp* __restrict__ ops,
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
  double2* st0 = wacc + nwarps * d.nslots;                // shared tiles (multi-segment passes)
  double2* st1 = st0 + (1u << d.k);
  for (int i = threadIdx.x; i < nwarps * d.nslots; i += nthr) wacc[i] = make_double2(0.0, 0.0);
  if (threadIdx.x < kMaxQubits) sq[threadIdx.x] = d.q[threadIdx.x];
  __syncthreads();

  const uint32_t tbase = uint32_t(lane) | (uint32_t(warp) << (5 + R));
  double2 v[NR], l[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) l[j] = make_double2(0.0, 0.0);
  const uint64_t ntiles = 1ull << (d.n - d.k);
  for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
    const uint64_t base = pdep64(T, d.rest);
    Map<R> m;
    make_map<R>(m, segs[d.seg_begin], sq, warp, wbits);
    load_g<R>(v, b0, base | lane | m.gw, m);
    if (NB == 2) load_g<R>(l, b1, base | lane | m.gw, m);
    bool in_smem = false;
    for (int s = d.seg_begin; s < d.seg_end; ++s) {
      const SegDesc sg = segs[s];
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
        for (int o = sg.op_begin; o < sg.op_end; ++o) {
          const RegOp op = rops[o];
          if ((base & op.co) != op.co) continue;
          const int sb = par64(base & op.zo);
          double2 z = make_double2(0.0, 0.0), z2 = make_double2(0.0, 0.0);
          if (op.kind == ROP_LAM) {
            if constexpr (NB == 2) pauli_op<R, 0>(l, v, op, tbase, sb, z, z2);
          } else if (NB == 1 || !(op.flags & RF_IP)) {
            pauli_op<R, 0>(v, l, op, tbase, sb, z, z2);
          } else if constexpr (NB == 2) {
            const uint32_t ipk = (op.flags >> 1) & 3u;
            if (op.flags & RF_IP_DIAG) {
              pauli_op<R, 3>(v, l, op, tbase, sb, z, z2);
            } else if (ipk == 1) {
              pauli_op<R, 1>(v, l, op, tbase, sb, z, z2);
            } else if (ipk == 2) {
              pauli_op<R, 2>(v, l, op, tbase, sb, z, z2);
            } else {
              pauli_op<R, 3>(v, l, op, tbase, sb, z, z2);
            }
            z = warp_sum(z);
            z2 = warp_sum(z2);
            if (lane == 0) {
              const double2 c = cfma(op.kb, z, cmul(op.ka, z2));
              double2& acc = wacc[warp * d.nslots + op.slot];
              acc = make_double2(acc.x + c.x, acc.y + c.y);
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
          if ((base & op.co) != op.co) continue;
          if (op.kind <= OP_APPLY_MAT2) {
            tile_apply(op.buf ? st1 : st0, d.k, op, coef + op.coef, base);
          } else {
            const double2 val = warp_sum(tile_ip(st0, st1, d.k, op, coef + op.coef, base));
            if (lane == 0) {
              double2& acc = wacc[warp * d.nslots + op.slot];
              acc = make_double2(acc.x + val.x, acc.y + val.y);
            }
          }
          __syncthreads();
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
    partials[d.part_off + static_cast<int64_t>(s) * gridDim.x + blockIdx.x] = acc;
  }
}

template __global__ void k_pass_reg<kRegBits, 1>(double2*, double2*, const PassDesc, const SegDesc*, const RegOp*,
                                                 const DevOp*, const double2*, double2*);
template __global__ void k_pass_reg<kRegBits, 2>(double2*, double2*, const PassDesc, const SegDesc*, const RegOp*,
                                                 const DevOp*, const double2*, double2*);

size_t reg_smem(int k, int nb, int nwarps, int nslots, bool tiles) {
  return sizeof(double2) * (size_t(nwarps) * nslots + (tiles ? (size_t(nb) << k) : 0));
}

static cudaError_t allow_dynamic_smem(const void* fn, size_t max_smem) {
  cudaFuncAttributes attr;
  cudaError_t e = cudaFuncGetAttributes(&attr, fn);
  if (e != cudaSuccess) return e;
  const size_t room = max_smem > attr.sharedSizeBytes ? max_smem - attr.sharedSizeBytes : 0;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(room));
}

cudaError_t prepare_reg_kernels(size_t max_smem) {
  cudaError_t e = allow_dynamic_smem(reinterpret_cast<const void*>(k_pass_reg<kRegBits, 1>), max_smem);
  if (e != cudaSuccess) return e;
  return allow_dynamic_smem(reinterpret_cast<const void*>(k_pass_reg<kRegBits, 2>), max_smem);
}

int reg_occupancy(int nb, int threads, size_t smem) {
  int blocks = 0;
  const void* fn = nb == 1 ? reinterpret_cast<const void*>(k_pass_reg<kRegBits, 1>)
                           : reinterpret_cast<const void*>(k_pass_reg<kRegBits, 2>);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, threads, smem);
  return blocks < 1 ? 1 : blocks;
}

void launch_pass_reg(int nb, const PassDesc& d, int grid, int threads, size_t smem, cudaStream_t s, double2* b0,
                     double2* b1, const SegDesc* segs, const RegOp* rops, const DevOp* ops, const double2* coef,
                     double2* partials) {
  if (nb == 1)
    k_pass_reg<kRegBits, 1><<<grid, threads, smem, s>>>(b0, b1, d, segs, rops, ops, coef, partials);
  else
    k_pass_reg<kRegBits, 2><<<grid, threads, smem, s>>>(b0, b1, d, segs, rops, ops, coef, partials);
}

}  // namespace svgb
