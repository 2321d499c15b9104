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

#include <algorithm>

#include "device.cuh"
#include "kernels.h"
#include "tile_ops.cuh"

namespace svgb {

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
    const uint64_t sbase = base | d.rank_bits;  // physical index bits for Z-signs / controls
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) tile[t] = psi[gidx(base, t, hi, d.b)];
    __syncthreads();
    for (int o = d.op_begin; o < d.op_end; ++o) {
      const DevOp op = ops[o];
      if ((sbase & op.co) != op.co) continue;
      tile_apply(tile, d.k, op, coef + op.coef, sbase);
      __syncthreads();
    }
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) psi[gidx(base, t, hi, d.b)] = tile[t];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) k_obs_pass(const double2* __restrict__ psi,
                                                       const double2* __restrict__ src_state,
                                                       double2* __restrict__ lam, PassDesc d,
                                                       const DevTerm* __restrict__ terms,
                                                       double2* __restrict__ partials) {
  // src_state: the shard whose amplitudes feed this pass's terms (== psi unless the
  // terms flip rank bits, d.xglob != 0: then the partner shard, fetched or peer-mapped).
  // The host sorts a pass's terms by tile flip mask: terms sharing a flip share
  // the partner amplitude, their signed coefficients are summed first.
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << d.k;
  const int nt = d.op_end - d.op_begin;
  const bool remote = d.xglob != 0;
  double2* tile = reinterpret_cast<double2*>(smem_raw);
  double2* wsum = tile + N;
  double2* cz = wsum + kWarps;                                   // [nt] coefficients, tile-uniform sign folded
  uint32_t* txl = reinterpret_cast<uint32_t*>(cz + nt);          // [nt] flip masks
  const int ne = (nt + 1) & ~1;                                  // keeps hi[] 8-byte aligned
  uint32_t* tzl = txl + ne;                                      // [nt] tile sign masks
  uint64_t* hi = reinterpret_cast<uint64_t*>(tzl + ne);
  build_hi(hi, d);
  for (int j = threadIdx.x; j < nt; j += blockDim.x) {
    txl[j] = terms[d.op_begin + j].xl;
    tzl[j] = terms[d.op_begin + j].zl;
  }
  double2 e = make_double2(0.0, 0.0);
  const uint64_t ntiles = 1ull << (d.n - d.k);
  for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
    const uint64_t base = pdep64(T, d.rest);
    const uint64_t sbase = base | d.rank_bits;  // physical index bits for Z-signs / controls
    const uint64_t src_bits = sbase ^ d.xglob;  // non-tile bits of the source amplitude index
    __syncthreads();  // previous tile done with tile[] / cz[]
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
      const DevTerm tm = terms[d.op_begin + j];
      cz[j] = cneg_if(tm.c, par64(src_bits & tm.zo));
    }
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) tile[t] = src_state[gidx(base, t, hi, d.b)];
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) {
      double2 acc = make_double2(0.0, 0.0);
      for (int j = 0; j < nt;) {
        const uint32_t xl = txl[j];
        const uint32_t src = t ^ xl;
        double2 cs = make_double2(0.0, 0.0);
        do {
          const double2 c = cneg_if(cz[j], par32(src & tzl[j]));
          cs = make_double2(cs.x + c.x, cs.y + c.y);
          ++j;
        } while (j < nt && txl[j] == xl);
        acc = cfma(cs, tile[src], acc);
      }
      const uint64_t m = gidx(base, t, hi, d.b);
      if (d.accumulate) {
        const double2 old = lam[m];
        lam[m] = make_double2(old.x + acc.x, old.y + acc.y);
      } else {
        lam[m] = acc;
      }
      e = cjfma(remote ? psi[m] : tile[t], acc, e);
    }
  }
  e = warp_sum(e);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 s = make_double2(0.0, 0.0);
    for (int w = 0; w < kWarps; ++w) s = make_double2(s.x + wsum[w].x, s.y + wsum[w].y);
    partials[d.part_off + blockIdx.x] = s;
  }
}

// Product-term pass (observable terms kept as products of 2x2 factors, e.g. the
// letters H / + / - of hadamard_all; svgrad/observable.py:79-100 applies them
// factor by factor with apply_matrix): the tile of `src` goes through this
// pass's factors as butterflies in shared memory, then either to `dst` (the
// product buffer, read by the next pass of the pipeline) or, on the last pass,
// into lambda as scalar * tile with the energy partial <psi | scalar * tile>.
__global__ void __launch_bounds__(kThreads) k_prod_pass(const double2* __restrict__ src, double2* __restrict__ dst,
                                                        const double2* __restrict__ psi, double2* __restrict__ lam,
                                                        PassDesc d, const __grid_constant__ ProdFactors f,
                                                        double2 scalar, double2* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << d.k;
  double2* tile = reinterpret_cast<double2*>(smem_raw);
  double2* wsum = tile + N;
  uint64_t* hi = reinterpret_cast<uint64_t*>(wsum + kWarps);
  build_hi(hi, d);
  double2 e = make_double2(0.0, 0.0);
  const uint64_t ntiles = 1ull << (d.n - d.k);
  for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
    const uint64_t base = pdep64(T, d.rest);
    __syncthreads();  // previous tile written out
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) tile[t] = src[gidx(base, t, hi, d.b)];
    __syncthreads();
    for (int j = 0; j < f.n; ++j) {
      const uint32_t pos = f.pos[j];
      const double2 m0 = f.m[j][0], m1 = f.m[j][1], m2 = f.m[j][2], m3 = f.m[j][3];
      for (uint32_t i = threadIdx.x; i < N / 2; i += blockDim.x) {
        const uint32_t i0 = insert0(i, pos), i1 = i0 | (1u << pos);
        const double2 v0 = tile[i0], v1 = tile[i1];
        tile[i0] = cfma(m1, v1, cmul(m0, v0));
        tile[i1] = cfma(m3, v1, cmul(m2, v0));
      }
      __syncthreads();
    }
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) {
      const uint64_t m = gidx(base, t, hi, d.b);
      if (!f.last) {
        dst[m] = tile[t];
        continue;
      }
      const double2 val = cmul(scalar, tile[t]);
      if (d.accumulate) {
        const double2 old = lam[m];
        lam[m] = make_double2(old.x + val.x, old.y + val.y);
      } else {
        lam[m] = val;
      }
      e = cjfma(psi[m], val, e);
    }
  }
  e = warp_sum(e);
  __syncthreads();
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
                                                         const double2* __restrict__ src_state,
                                                         double2* __restrict__ lam, PassDesc d,
                                                         const DevTerm* __restrict__ terms,
                                                         double2* __restrict__ partials) {
  __shared__ double2 wsum[kWarps];
  double2 e = make_double2(0.0, 0.0);
  const uint64_t dim = 1ull << d.n;
  const uint64_t src_bits = d.rank_bits ^ d.xglob;  // rank bits of the source amplitude index
  for (uint64_t m = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; m < dim; m += uint64_t(gridDim.x) * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = d.op_begin; j < d.op_end; ++j) {
      const DevTerm tm = terms[j];
      const uint64_t x = uint64_t(tm.xl) | (uint64_t(tm.zl) << 32);  // local part of the flip mask
      const uint64_t src = m ^ x;
      acc = cfma(cneg_if(tm.c, par64((src | src_bits) & tm.zo)), src_state[src], acc);
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
    const uint64_t sbase = base | d.rank_bits;  // physical index bits for Z-signs / controls
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) {
      const uint64_t m = gidx(base, t, hi, d.b);
      tp[t] = phi[m];
      tl[t] = lam[m];
    }
    __syncthreads();
    for (int o = d.op_begin; o < d.op_end; ++o) {
      const DevOp op = ops[o];
      if ((sbase & op.co) != op.co) continue;
      if (op.kind <= OP_APPLY_MAT2) {
        tile_apply(op.buf ? tl : tp, d.k, op, coef + op.coef, sbase);
      } else {
        const double2 v = warp_sum(tile_ip(tp, tl, d.k, op, coef + op.coef, sbase));
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

// One warp per sum: lane l adds partials l, l+32, ... in order, then a fixed
// shuffle tree -- the same order on every run (deterministic), 32x the
// memory-level parallelism of a thread per sum.
__global__ void k_finalize(const double2* __restrict__ partials, const SumSpec* __restrict__ specs,
                           int count, double2* __restrict__ out) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= count) return;
  const SumSpec sp = specs[i];
  // four independent accumulators (loads in flight together); the order of the
  // additions is fixed by (lane, count), so reruns stay bit-identical
  double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
  const double2* p = partials + sp.off;
  int64_t c = lane;
  for (; c + 96 < sp.count; c += 128) {
    const double2 v0 = p[c], v1 = p[c + 32], v2 = p[c + 64], v3 = p[c + 96];
    a0 = make_double2(a0.x + v0.x, a0.y + v0.y);
    a1 = make_double2(a1.x + v1.x, a1.y + v1.y);
    a2 = make_double2(a2.x + v2.x, a2.y + v2.y);
    a3 = make_double2(a3.x + v3.x, a3.y + v3.y);
  }
  for (; c < sp.count; c += 32) {
    const double2 v = p[c];
    a0 = make_double2(a0.x + v.x, a0.y + v.y);
  }
  double2 acc = make_double2((a0.x + a1.x) + (a2.x + a3.x), (a0.y + a1.y) + (a2.y + a3.y));
  acc = warp_sum(acc);
  if (lane == 0) out[i] = acc;
}

__global__ void k_set_basis(double2* psi, uint64_t idx) { psi[idx] = make_double2(1.0, 0.0); }

// Qubit swap between rank bit `gbit` and local bit `lpos` (virtual shards in one
// allocation).  Amplitude (rank r, local m) with r_g = a, m_p = c moves to
// (r with r_g = c, m with m_p = a): shard pairs exchange lower[m | p] <-> upper[m].
__global__ void k_swap_virtual(double2* __restrict__ state, int nloc, int nshards, int gbit, int lpos) {
  const uint64_t half = 1ull << (nloc - 1);
  const uint64_t pairs = uint64_t(nshards / 2) * half;
  const uint64_t pbit = 1ull << lpos;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < pairs; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t pr = i >> (nloc - 1), m0 = i & (half - 1);
    const uint64_t lo_rank = ((pr >> gbit) << (gbit + 1)) | (pr & ((1ull << gbit) - 1));  // rank bit gbit = 0
    const uint64_t hi_rank = lo_rank | (1ull << gbit);
    const uint64_t m = ((m0 >> lpos) << (lpos + 1)) | (m0 & (pbit - 1));  // local bit lpos = 0
    double2* a = state + (lo_rank << nloc) + (m | pbit);
    double2* b = state + (hi_rank << nloc) + m;
    const double2 t = *a;
    *a = *b;
    *b = t;
  }
}

// packed[i] = shard[i with bit lpos inserted = val]   (and the inverse scatter)
__global__ void k_half_pack(const double2* __restrict__ shard, double2* __restrict__ packed, int nloc, int lpos,
                            int val, int unpack) {
  const uint64_t half = 1ull << (nloc - 1);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < half; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t m = ((i >> lpos) << (lpos + 1)) | (i & ((1ull << lpos) - 1)) | (uint64_t(val) << lpos);
    if (unpack)
      const_cast<double2*>(shard)[m] = packed[i];
    else
      packed[i] = shard[m];
  }
}

// ------------------------------------------------------------ launchers --

size_t fwd_smem(int k, int b) { return (sizeof(double2) << k) + (sizeof(uint64_t) << (k - b)); }
size_t obs_smem(int k, int b, int nterms) {
  return (sizeof(double2) << k) + sizeof(double2) * kWarps + sizeof(double2) * nterms +
         sizeof(uint32_t) * 2 * ((nterms + 1) & ~1) + (sizeof(uint64_t) << (k - b));
}
size_t prod_smem(int k, int b) {
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
  if ((e = set_smem_attr(reinterpret_cast<const void*>(k_prod_pass), max_smem)) != cudaSuccess) return e;
  return set_smem_attr(reinterpret_cast<const void*>(k_rev_pass), max_smem);
}

int occupancy(int which, size_t smem) {
  int blocks = 0;
  const void* fn = which == 0 ? reinterpret_cast<const void*>(k_fwd_pass)
                 : which == 1 ? reinterpret_cast<const void*>(k_obs_pass)
                 : which == 3 ? reinterpret_cast<const void*>(k_prod_pass)
                              : reinterpret_cast<const void*>(k_rev_pass);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kThreads, smem);
  return blocks < 1 ? 1 : blocks;
}

void launch_fwd(const PassDesc& d, int grid, size_t smem, cudaStream_t s, double2* psi,
                const DevOp* ops, const double2* coef) {
  k_fwd_pass<<<grid, kThreads, smem, s>>>(psi, d, ops, coef);
}
void launch_obs(const PassDesc& d, int grid, size_t smem, cudaStream_t s, const double2* psi, const double2* src,
                double2* lam, const DevTerm* terms, double2* partials) {
  k_obs_pass<<<grid, kThreads, smem, s>>>(psi, src, lam, d, terms, partials);
}
void launch_prod(const PassDesc& d, const ProdFactors& f, int grid, size_t smem, cudaStream_t s, const double2* src,
                 double2* dst, const double2* psi, double2* lam, double2 scalar, double2* partials) {
  k_prod_pass<<<grid, kThreads, smem, s>>>(src, dst, psi, lam, d, f, scalar, partials);
}
void launch_obs_direct(const PassDesc& d, int grid, cudaStream_t s, const double2* psi, const double2* src,
                       double2* lam, const DevTerm* terms, double2* partials) {
  k_obs_direct<<<grid, kThreads, 0, s>>>(psi, src, lam, d, terms, partials);
}
void launch_rev(const PassDesc& d, int grid, size_t smem, cudaStream_t s, double2* phi, double2* lam,
                const DevOp* ops, const double2* coef, double2* partials) {
  k_rev_pass<<<grid, kThreads, smem, s>>>(phi, lam, d, ops, coef, partials);
}
void launch_finalize(const double2* partials, const SumSpec* specs, int count, double2* out,
                     cudaStream_t s) {
  if (count <= 0) return;
  k_finalize<<<(count + 3) / 4, 128, 0, s>>>(partials, specs, count, out);  // 4 sums (warps) per block
}
void launch_set_basis(double2* psi, uint64_t idx, cudaStream_t s) { k_set_basis<<<1, 1, 0, s>>>(psi, idx); }

static int stream_grid(uint64_t items) {
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((items + 255) / 256, 148ull * 16)));
}
void launch_swap_virtual(double2* state, int nloc, int nshards, int gbit, int lpos, cudaStream_t s) {
  const uint64_t pairs = uint64_t(nshards / 2) << (nloc - 1);
  k_swap_virtual<<<stream_grid(pairs), 256, 0, s>>>(state, nloc, nshards, gbit, lpos);
}
void launch_half_pack(const double2* shard, double2* packed, int nloc, int lpos, int val, cudaStream_t s) {
  k_half_pack<<<stream_grid(1ull << (nloc - 1)), 256, 0, s>>>(shard, packed, nloc, lpos, val, 0);
}
void launch_half_unpack(const double2* packed, double2* shard, int nloc, int lpos, int val, cudaStream_t s) {
  k_half_pack<<<stream_grid(1ull << (nloc - 1)), 256, 0, s>>>(shard, const_cast<double2*>(packed), nloc, lpos, val, 1);
}

}  // namespace svgb
