// Device helpers shared by the shared-memory tile kernels (kernels.cu) and the
// register-tile kernels (kernels_reg.cu): complex arithmetic, bit tricks, and
// the generic tile-local gate/inner-product ops on a shared-memory tile.
#pragma once
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#endif

#include "device.cuh"

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
__device__ inline void build_hi(uint64_t* hi, const PassDesc& d) {
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

__device__ inline void tile_apply(double2* s, int k, const DevOp& op, const double2* cf, uint64_t base) {
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
__device__ inline double2 tile_ip(const double2* phi, const double2* lam, int k, const DevOp& op,
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

}  // namespace svgb
