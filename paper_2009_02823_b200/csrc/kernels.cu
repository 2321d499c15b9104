// Tile-pass kernels for sm_100a (v1: shared-memory tiles, one CTA per tile at a time).
//
//   k_fwd_pass  -- K1: psi <- U_b..U_a psi for every gate of a pass, one HBM
//                  read+write of psi per pass          (svgrad/gradients.py:149-150)
//   k_obs_pass  -- K2: lambda (+)= sum_t c_t P_t psi over the pass's Pauli
//                  strings, fused with the energy partial <psi|lambda>
//                                                       (svgrad/observable.py:79-100,
//                                                        svgrad/gradients.py:153-156)
//   k_rev_pass  -- K3: per gate (descending): phi <- R phi; slot += <lam|K|phi>;
//                  lam <- U^dag lam.  mu (the probe) is never materialised
//                                                       (svgrad/gradients.py:158-168)
//   k_finalize  -- K4: deterministic fixed-order sums of the per-CTA partials
//
// Every reduction is per-warp shuffle -> per-(warp,slot) shared accumulator ->
// fixed-order per-CTA sum -> fixed-order cross-CTA sum: no atomics, so a
// rerun is bit-identical.
#include <cuda_runtime.h>

#include "device.cuh"
#include "kernels.h"

namespace svgb {

// ---------------------------------------------------------------- helpers --

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a*b + c
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// conj(a)*b + c
__device__ __forceinline__ double2 cjfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 cneg_if(double2 a, int s) {
  return s ? make_double2(-a.x, -a.y) : a;
}
__device__ __forceinline__ int par32(uint32_t v) { return __popc(v) & 1; }
__device__ __forceinline__ int par64(uint64_t v) { return __popcll(v) & 1; }
__device__ __forceinline__ uint32_t insert0(uint32_t p, int pos) {
  return ((p >> pos) << (pos + 1)) | (p & ((1u << pos) - 1u));
}
// Scatter the low bits of v into the set bits of mask (software PDEP).
__device__ __forceinline__ uint64_t pdep64(uint64_t v, uint64_t mask) {
  uint64_t r = 0;
  for (uint64_t bit = 1; mask; bit <<= 1) {
    const uint64_t low = mask & (~mask + 1);
    if (v & bit) r |= low;
    mask &= mask - 1;
  }
  return r;
}
__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// hi[i] = global offset of tile-local index (i << b)
__device__ void build_hi(uint64_t* hi, const PassDesc& d) {
  const int nh = 1 << (d.k - d.b);
  for (int i = threadIdx.x; i < nh; i += blockDim.x) {
    uint64_t off = 0;
    for (int j = d.b; j < d.k; ++j)
      if ((i >> (j - d.b)) & 1) off |= 1ull << d.q[j];
    hi[i] = off;
  }
}
__device__ __forceinline__ uint64_t gidx(uint64_t base, uint32_t t, const uint64_t* hi, int b) {
  return base | (t & ((1u << b) - 1u)) | hi[t >> b];
}

// ------------------------------------------------------------ tile ops --

__device__ void tile_apply(double2* s, int k, const DevOp& op, const double2* cf, uint64_t base) {
  const uint32_t N = 1u << k;
  const uint32_t cl = op.cl;
  if (op.kind == OP_APPLY_PAULI) {
    const double2 a = cf[0], bb = cf[1];
    const int sb = par64(base & op.zo);
    if (op.xl == 0) {
      const double2 fp = make_double2(a.x + bb.x, a.y + bb.y);
      const double2 fm = make_double2(a.x - bb.x, a.y - bb.y);
      for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) {
        if ((t & cl) != cl) continue;
        s[t] = cmul((par32(t & op.zl) ^ sb) ? fm : fp, s[t]);
      }
    } else {
      const int piv = __ffs(op.xl) - 1;
      for (uint32_t p = threadIdx.x; p < N / 2; p += blockDim.x) {
        const uint32_t t0 = insert0(p, piv), t1 = t0 ^ op.xl;
        if ((t0 & cl) != cl) continue;
        const double2 v0 = s[t0], v1 = s[t1];
        const int s0 = par32(t0 & op.zl) ^ sb, s1 = par32(t1 & op.zl) ^ sb;
        s[t0] = cfma(cneg_if(bb, s1), v1, cmul(a, v0));
        s[t1] = cfma(cneg_if(bb, s0), v0, cmul(a, v1));
      }
    }
  } else if (op.kind == OP_APPLY_MAT1) {
    const double2 m0 = cf[0], m1 = cf[1], m2 = cf[2], m3 = cf[3];
    for (uint32_t p = threadIdx.x; p < N / 2; p += blockDim.x) {
      const uint32_t i0 = insert0(p, op.t0), i1 = i0 | (1u << op.t0);
      if ((i0 & cl) != cl) continue;
      const double2 v0 = s[i0], v1 = s[i1];
      s[i0] = cfma(m1, v1, cmul(m0, v0));
      s[i1] = cfma(m3, v1, cmul(m2, v0));
    }
  } else {  // OP_APPLY_MAT2
    const int lo = min(op.t0, op.t1), hi = max(op.t0, op.t1);
    for (uint32_t p = threadIdx.x; p < N / 4; p += blockDim.x) {
      const uint32_t i = insert0(insert0(p, lo), hi);
      if ((i & cl) != cl) continue;
      uint32_t idx[4];
      double2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        idx[q] = i | ((q & 1u) << op.t0) | ((q >> 1) << op.t1);
        v[q] = s[idx[q]];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double2 acc = cmul(cf[4 * r], v[0]);
        acc = cfma(cf[4 * r + 1], v[1], acc);
        acc = cfma(cf[4 * r + 2], v[2], acc);
        acc = cfma(cf[4 * r + 3], v[3], acc);
        s[idx[r]] = acc;
      }
    }
  }
}

// <lam| K |phi> restricted to this thread's share of the tile.
__device__ double2 tile_ip(const double2* phi, const double2* lam, int k, const DevOp& op,
                           const double2* cf, uint64_t base) {
  const uint32_t N = 1u << k;
  const uint32_t cl = op.cl;
  double2 acc = make_double2(0.0, 0.0);
  if (op.kind == OP_IP_PAULI) {
    const double2 ka = cf[0], kb = cf[1];
    const int sb = par64(base & op.zo);
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) {
      if ((t & cl) != cl) continue;
      const uint32_t j = t ^ op.xl;
      const double2 kv = cfma(cneg_if(kb, par32(j & op.zl) ^ sb), phi[j], cmul(ka, phi[t]));
      acc = cjfma(lam[t], kv, acc);
    }
  } else if (op.kind == OP_IP_MAT1) {
    const double2 m0 = cf[0], m1 = cf[1], m2 = cf[2], m3 = cf[3];
    for (uint32_t p = threadIdx.x; p < N / 2; p += blockDim.x) {
      const uint32_t i0 = insert0(p, op.t0), i1 = i0 | (1u << op.t0);
      if ((i0 & cl) != cl) continue;
      const double2 v0 = phi[i0], v1 = phi[i1];
      acc = cjfma(lam[i0], cfma(m1, v1, cmul(m0, v0)), acc);
      acc = cjfma(lam[i1], cfma(m3, v1, cmul(m2, v0)), acc);
    }
  } else {  // OP_IP_MAT2
    const int lo = min(op.t0, op.t1), hi = max(op.t0, op.t1);
    for (uint32_t p = threadIdx.x; p < N / 4; p += blockDim.x) {
      const uint32_t i = insert0(insert0(p, lo), hi);
      if ((i & cl) != cl) continue;
      uint32_t idx[4];
      double2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        idx[q] = i | ((q & 1u) << op.t0) | ((q >> 1) << op.t1);
        v[q] = phi[idx[q]];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double2 kv = cmul(cf[4 * r], v[0]);
        kv = cfma(cf[4 * r + 1], v[1], kv);
        kv = cfma(cf[4 * r + 2], v[2], kv);
        kv = cfma(cf[4 * r + 3], v[3], kv);
        acc = cjfma(lam[idx[r]], kv, acc);
      }
    }
  }
  return acc;
}

// ------------------------------------------------------------ kernels --

__global__ void __launch_bounds__(kThreads) k_fwd_pass(double2* __restrict__ psi, PassDesc d,
                                                       const DevOp* __restrict__ ops,
                                                       const double2* __restrict__ coef) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << d.k;
  double2* tile = reinterpret_cast<double2*>(smem_raw);
  uint64_t* hi = reinterpret_cast<uint64_t*>(tile + N);
  build_hi(hi, d);
  __syncthreads();
  const uint64_t ntiles = 1ull << (d.n - d.k);
  for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
    const uint64_t base = pdep64(T, d.rest);
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) tile[t] = psi[gidx(base, t, hi, d.b)];
    __syncthreads();
    for (int o = d.op_begin; o < d.op_end; ++o) {
      const DevOp op = ops[o];
      if ((base & op.co) != op.co) continue;
      tile_apply(tile, d.k, op, coef + op.coef, base);
      __syncthreads();
    }
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) psi[gidx(base, t, hi, d.b)] = tile[t];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) k_obs_pass(const double2* __restrict__ psi,
                                                       double2* __restrict__ lam, PassDesc d,
                                                       const DevTerm* __restrict__ terms,
                                                       double2* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << d.k;
  double2* tile = reinterpret_cast<double2*>(smem_raw);
  double2* wsum = tile + N;
  uint64_t* hi = reinterpret_cast<uint64_t*>(wsum + kWarps);
  build_hi(hi, d);
  __syncthreads();
  double2 e = make_double2(0.0, 0.0);
  const uint64_t ntiles = 1ull << (d.n - d.k);
  for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
    const uint64_t base = pdep64(T, d.rest);
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) tile[t] = psi[gidx(base, t, hi, d.b)];
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) {
      double2 acc = make_double2(0.0, 0.0);
      for (int j = d.op_begin; j < d.op_end; ++j) {
        const DevTerm tm = terms[j];
        const uint32_t src = t ^ tm.xl;
        const int sg = par32(src & tm.zl) ^ par64(base & tm.zo);
        acc = cfma(cneg_if(tm.c, sg), tile[src], acc);
      }
      const uint64_t m = gidx(base, t, hi, d.b);
      if (d.accumulate) {
        const double2 old = lam[m];
        lam[m] = make_double2(old.x + acc.x, old.y + acc.y);
      } else {
        lam[m] = acc;
      }
      e = cjfma(tile[t], acc, e);
    }
    __syncthreads();
  }
  e = warp_sum(e);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 s = make_double2(0.0, 0.0);
    for (int w = 0; w < kWarps; ++w) s = make_double2(s.x + wsum[w].x, s.y + wsum[w].y);
    partials[d.part_off + blockIdx.x] = s;
  }
}

// Untiled observable pass for flip masks too wide for a tile: plain gathers.
__global__ void __launch_bounds__(kThreads) k_obs_direct(const double2* __restrict__ psi,
                                                         double2* __restrict__ lam, PassDesc d,
                                                         const DevTerm* __restrict__ terms,
                                                         double2* __restrict__ partials) {
  __shared__ double2 wsum[kWarps];
  double2 e = make_double2(0.0, 0.0);
  const uint64_t dim = 1ull << d.n;
  for (uint64_t m = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; m < dim; m += uint64_t(gridDim.x) * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = d.op_begin; j < d.op_end; ++j) {
      const DevTerm tm = terms[j];
      const uint64_t x = uint64_t(tm.xl) | (uint64_t(tm.zl) << 32);
      const uint64_t src = m ^ x;
      acc = cfma(cneg_if(tm.c, par64(src & tm.zo)), psi[src], acc);
    }
    if (d.accumulate) {
      const double2 old = lam[m];
      lam[m] = make_double2(old.x + acc.x, old.y + acc.y);
    } else {
      lam[m] = acc;
    }
    e = cjfma(psi[m], acc, e);
  }
  e = warp_sum(e);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 s = make_double2(0.0, 0.0);
    for (int w = 0; w < kWarps; ++w) s = make_double2(s.x + wsum[w].x, s.y + wsum[w].y);
    partials[d.part_off + blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kThreads) k_rev_pass(double2* __restrict__ phi,
                                                       double2* __restrict__ lam, PassDesc d,
                                                       const DevOp* __restrict__ ops,
                                                       const double2* __restrict__ coef,
                                                       double2* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << d.k;
  double2* tp = reinterpret_cast<double2*>(smem_raw);
  double2* tl = tp + N;
  double2* wacc = tl + N;  // [kWarps][nslots]
  uint64_t* hi = reinterpret_cast<uint64_t*>(wacc + kWarps * d.nslots);
  build_hi(hi, d);
  for (int i = threadIdx.x; i < kWarps * d.nslots; i += blockDim.x) wacc[i] = make_double2(0.0, 0.0);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t ntiles = 1ull << (d.n - d.k);
  for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
    const uint64_t base = pdep64(T, d.rest);
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) {
      const uint64_t m = gidx(base, t, hi, d.b);
      tp[t] = phi[m];
      tl[t] = lam[m];
    }
    __syncthreads();
    for (int o = d.op_begin; o < d.op_end; ++o) {
      const DevOp op = ops[o];
      if ((base & op.co) != op.co) continue;
      if (op.kind <= OP_APPLY_MAT2) {
        tile_apply(op.buf ? tl : tp, d.k, op, coef + op.coef, base);
      } else {
        const double2 v = warp_sum(tile_ip(tp, tl, d.k, op, coef + op.coef, base));
        if (lane == 0) {
          double2& a = wacc[warp * d.nslots + op.slot];
          a = make_double2(a.x + v.x, a.y + v.y);
        }
      }
      __syncthreads();
    }
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) {
      const uint64_t m = gidx(base, t, hi, d.b);
      phi[m] = tp[t];
      lam[m] = tl[t];
    }
    __syncthreads();
  }
  for (int s = threadIdx.x; s < d.nslots; s += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int w = 0; w < kWarps; ++w) {
      const double2 v = wacc[w * d.nslots + s];
      acc = make_double2(acc.x + v.x, acc.y + v.y);
    }
    partials[d.part_off + static_cast<int64_t>(s) * gridDim.x + blockIdx.x] = acc;
  }
}

__global__ void k_finalize(const double2* __restrict__ partials, const SumSpec* __restrict__ specs,
                           int count, double2* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const SumSpec sp = specs[i];
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t c = 0; c < sp.count; ++c) {
    const double2 v = partials[sp.off + c];
    acc = make_double2(acc.x + v.x, acc.y + v.y);
  }
  out[i] = acc;
}

__global__ void k_set_basis(double2* psi, uint64_t idx) { psi[idx] = make_double2(1.0, 0.0); }

// ------------------------------------------------------------ launchers --

size_t fwd_smem(int k, int b) { return (sizeof(double2) << k) + (sizeof(uint64_t) << (k - b)); }
size_t obs_smem(int k, int b) {
  return (sizeof(double2) << k) + sizeof(double2) * kWarps + (sizeof(uint64_t) << (k - b));
}
size_t rev_smem(int k, int b, int nslots) {
  return (2 * sizeof(double2) << k) + sizeof(double2) * kWarps * nslots + (sizeof(uint64_t) << (k - b));
}

static cudaError_t set_smem_attr(const void* fn, size_t bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

cudaError_t prepare_kernels(size_t max_smem) {
  cudaError_t e;
  if ((e = set_smem_attr(reinterpret_cast<const void*>(k_fwd_pass), max_smem)) != cudaSuccess) return e;
  if ((e = set_smem_attr(reinterpret_cast<const void*>(k_obs_pass), max_smem)) != cudaSuccess) return e;
  return set_smem_attr(reinterpret_cast<const void*>(k_rev_pass), max_smem);
}

int occupancy(int which, size_t smem) {
  int blocks = 0;
  const void* fn = which == 0 ? reinterpret_cast<const void*>(k_fwd_pass)
                 : which == 1 ? reinterpret_cast<const void*>(k_obs_pass)
                              : reinterpret_cast<const void*>(k_rev_pass);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kThreads, smem);
  return blocks < 1 ? 1 : blocks;
}

void launch_fwd(const PassDesc& d, int grid, size_t smem, cudaStream_t s, double2* psi,
                const DevOp* ops, const double2* coef) {
  k_fwd_pass<<<grid, kThreads, smem, s>>>(psi, d, ops, coef);
}
void launch_obs(const PassDesc& d, int grid, size_t smem, cudaStream_t s, const double2* psi,
                double2* lam, const DevTerm* terms, double2* partials) {
  k_obs_pass<<<grid, kThreads, smem, s>>>(psi, lam, d, terms, partials);
}
void launch_obs_direct(const PassDesc& d, int grid, cudaStream_t s, const double2* psi, double2* lam,
                       const DevTerm* terms, double2* partials) {
  k_obs_direct<<<grid, kThreads, 0, s>>>(psi, lam, d, terms, partials);
}
void launch_rev(const PassDesc& d, int grid, size_t smem, cudaStream_t s, double2* phi, double2* lam,
                const DevOp* ops, const double2* coef, double2* partials) {
  k_rev_pass<<<grid, kThreads, smem, s>>>(phi, lam, d, ops, coef, partials);
}
void launch_finalize(const double2* partials, const SumSpec* specs, int count, double2* out,
                     cudaStream_t s) {
  if (count <= 0) return;
  k_finalize<<<(count + 127) / 128, 128, 0, s>>>(partials, specs, count, out);
}
void launch_set_basis(double2* psi, uint64_t idx, cudaStream_t s) { k_set_basis<<<1, 1, 0, s>>>(psi, idx); }

}  // namespace svgb
