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
#include "reg_ops.cuh"
#include "tile_ops.cuh"

namespace svgb {

namespace {

constexpr int kRegThreads = 256;  // launch bound: k = 11 tiles with R = 3 (8 warps)

template <int R, int NB, int V>
__device__ __forceinline__ void run_variant(double2 (&v)[1 << R], double2 (&l)[1 << R], const RegOp& op,
                                            const OpCtx& c, uint32_t slw, const IpSink& sink) {
  op_body<R, NB, V>(v, l, c, op.xl, slw, (op.flags & RF_BI) != 0, op.slot, op.kr, op.ka, op.kb, sink);
}

#define SVGB_V1(N) \
  case (N):        \
    run_variant<R, NB, (N)>(v, l, op, c, slw, sink); \
    break;
#define SVGB_V4(N) SVGB_V1(N) SVGB_V1(N + 1) SVGB_V1(N + 2) SVGB_V1(N + 3)
#define SVGB_V20(N) SVGB_V4(N) SVGB_V4(N + 4) SVGB_V4(N + 8) SVGB_V4(N + 12) SVGB_V4(N + 16)

// Dense switch over exactly the kernel's variants (a single jump table).
template <int R, int NB>
__device__ __forceinline__ void dispatch(uint32_t id, double2 (&v)[1 << R], double2 (&l)[1 << R], const RegOp& op,
                                         OpCtx& c, uint32_t slw, const IpSink& sink) {
  constexpr int NV = Pat<R>::N * 2 * (NB == 2 ? kRevModes : kFwdModes);
  static_assert(NV % 20 == 0 || NV % 4 == 0, "variant count");
  if constexpr (R == 4) {  // N = 20
    if constexpr (NB == 1) {
      static_assert(NV == 160, "");
      switch (id) {
        SVGB_V20(0) SVGB_V20(20) SVGB_V20(40) SVGB_V20(60) SVGB_V20(80) SVGB_V20(100) SVGB_V20(120) SVGB_V20(140)
        default: break;
      }
    } else {
      static_assert(NV == 200, "");
      switch (id) {
        SVGB_V20(0) SVGB_V20(20) SVGB_V20(40) SVGB_V20(60) SVGB_V20(80) SVGB_V20(100) SVGB_V20(120) SVGB_V20(140)
        SVGB_V20(160) SVGB_V20(180)
        default: break;
      }
    }
  } else {  // R == 3: N = 16
    if constexpr (NB == 1) {
      static_assert(NV == 128, "");
      switch (id) {
        SVGB_V4(0) SVGB_V4(4) SVGB_V4(8) SVGB_V4(12) SVGB_V4(16) SVGB_V4(20) SVGB_V4(24) SVGB_V4(28)
        SVGB_V4(32) SVGB_V4(36) SVGB_V4(40) SVGB_V4(44) SVGB_V4(48) SVGB_V4(52) SVGB_V4(56) SVGB_V4(60)
        SVGB_V4(64) SVGB_V4(68) SVGB_V4(72) SVGB_V4(76) SVGB_V4(80) SVGB_V4(84) SVGB_V4(88) SVGB_V4(92)
        SVGB_V4(96) SVGB_V4(100) SVGB_V4(104) SVGB_V4(108) SVGB_V4(112) SVGB_V4(116) SVGB_V4(120) SVGB_V4(124)
        default: break;
      }
    } else {
      static_assert(NV == 160, "");
      switch (id) {
        SVGB_V20(0) SVGB_V20(20) SVGB_V20(40) SVGB_V20(60) SVGB_V20(80) SVGB_V20(100) SVGB_V20(120) SVGB_V20(140)
        default: break;
      }
    }
  }
}
#undef SVGB_V20
#undef SVGB_V4
#undef SVGB_V1

}  // namespace

template <int R, int NB>
__global__ void __launch_bounds__(R == 3 ? kRegThreads : kRegThreads / 2, R == 3 ? 2 : (NB == 2 ? 2 : 4))
    k_pass_reg(double2* __restrict__ b0, double2* __restrict__ b1, const PassDesc d, const SegDesc* __restrict__ segs,
               const RegOp* __restrict__ rops, const DevOp* __restrict__ ops, const double2* __restrict__ coef,
               double2* __restrict__ partials) {
  constexpr int NR = 1 << R;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint8_t sq[kMaxQubits];
  const int nthr = blockDim.x;
  const int nwarps = nthr >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wbits = d.k - 5 - R;
  const int nsegs = d.seg_end - d.seg_begin;
  double2* wacc = reinterpret_cast<double2*>(smem_raw);  // [nwarps][nslots]
  SegDesc* ssegs = reinterpret_cast<SegDesc*>(wacc + nwarps * d.nslots);  // this pass's segments
  RegOp* sops = reinterpret_cast<RegOp*>(ssegs + nsegs);                  // this pass's register ops
  const int nops = d.op_end - d.op_begin;
  const int nacc = nthr >> d.acc_shift;  // accumulators per slot
  double* tacc = d.thread_acc ? reinterpret_cast<double*>(sops + nops) : nullptr;  // [nslots][nacc]
  double2* st0 = reinterpret_cast<double2*>(sops + nops) + (d.thread_acc ? (d.nslots * nacc + 1) / 2 : 0);
  double2* st1 = st0 + (1u << d.k);  // shared tiles (multi-segment passes)
  for (int i = threadIdx.x; i < nwarps * d.nslots; i += nthr) wacc[i] = make_double2(0.0, 0.0);
  if (tacc)
    for (int i = threadIdx.x; i < d.nslots * nacc; i += nthr) tacc[i] = 0.0;
  {
    const uint4* src = reinterpret_cast<const uint4*>(rops + d.op_begin);
    uint4* dst = reinterpret_cast<uint4*>(sops);
    for (int i = threadIdx.x; i < nops * int(sizeof(RegOp) / 16); i += nthr) dst[i] = src[i];
    const uint4* ssrc = reinterpret_cast<const uint4*>(segs + d.seg_begin);
    uint4* sdst = reinterpret_cast<uint4*>(ssegs);
    for (int i = threadIdx.x; i < nsegs * int(sizeof(SegDesc) / 16); i += nthr) sdst[i] = ssrc[i];
  }
  if (threadIdx.x < kMaxQubits) sq[threadIdx.x] = d.q[threadIdx.x];
  __syncthreads();
  const IpSink sink{tacc, wacc, nthr, d.nslots, warp, lane, d.acc_shift};

  const uint32_t tbase = uint32_t(lane) | (uint32_t(warp) << (5 + R));
  double2 v[NR], l[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) l[j] = make_double2(0.0, 0.0);
  const uint64_t ntiles = 1ull << (d.n - d.k);
  for (uint64_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
    const uint64_t base = pdep64(T, d.rest);
    const uint64_t sbase = base | d.rank_bits;  // physical index bits for Z-signs / controls
    int mseg = 0;  // segment whose register layout v / l are in
    {
      Map<R> m;
      make_map<R>(m, ssegs[0], sq, warp, wbits);
      load_g<R>(v, b0, base | lane | m.gw, m);
      if (NB == 2) load_g<R>(l, b1, base | lane | m.gw, m);
    }
    bool in_smem = false;
    double pend = 1.0;  // deferred scale of the register tile (see upd)
    for (int s = 0; s < nsegs; ++s) {
      const SegDesc& sg = ssegs[s];
      if (sg.kind == SEG_REG) {
        if (s != 0 && (in_smem || !sg.same_map)) {
          if (!in_smem) {
            if (pend != 1.0) {
              scale_tile<R>(v, pend);
              if (NB == 2) scale_tile<R>(l, pend);
            }
            __syncthreads();
            Map<R> m;
            make_map<R>(m, ssegs[mseg], sq, warp, wbits);
            to_smem<R>(v, st0, lane | m.sw, m);
            if (NB == 2) to_smem<R>(l, st1, lane | m.sw, m);
          }
          __syncthreads();
          mseg = s;
          Map<R> m;
          make_map<R>(m, sg, sq, warp, wbits);
          from_smem<R>(v, st0, lane | m.sw, m);
          if (NB == 2) from_smem<R>(l, st1, lane | m.sw, m);
          in_smem = false;
        }
        const RegOp* op_end = sops + (sg.op_end - d.op_begin);
        for (const RegOp* po = sops + (sg.op_begin - d.op_begin); po != op_end; ++po) {
          const RegOp& op = *po;
          if ((sbase & op.co) != op.co) continue;
          const uint32_t slw = uint32_t(__popc((tbase ^ op.xl) & op.zlw) ^ __popcll(sbase & op.zo)) & 1u;
          OpCtx c;
          c.a = op.a;
          c.bb = slw ? -op.bb : op.bb;  // uniform part of the partner sign
          c.smask = op.smask;
          c.cmask = op.cmask;
          c.clw_ok = (tbase & op.clw) == op.clw;
          c.pneg = c.bb < 0.0;
          dispatch<R, NB>(op.variant, v, l, op, c, slw, sink);
        }
        pend = sg.scale;
      } else {  // SEG_SMEM: generic dense-matrix ops on the shared-memory tile
        if (!in_smem) {
          if (pend != 1.0) {
            scale_tile<R>(v, pend);
            if (NB == 2) scale_tile<R>(l, pend);
            pend = 1.0;
          }
          __syncthreads();
          Map<R> m;
          make_map<R>(m, ssegs[mseg], sq, warp, wbits);
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
      }
    }
    Map<R> m;
    make_map<R>(m, ssegs[mseg], sq, warp, wbits);
    if (in_smem) {
      from_smem<R>(v, st0, lane | m.sw, m);
      if (NB == 2) from_smem<R>(l, st1, lane | m.sw, m);
    } else if (pend != 1.0) {
      scale_tile<R>(v, pend);
      if (NB == 2) scale_tile<R>(l, pend);
    }
    store_g<R>(v, b0, base | lane | m.gw, m);
    if (NB == 2) store_g<R>(l, b1, base | lane | m.gw, m);
  }
  if (d.nslots == 0) return;
  __syncthreads();
  flush_partials(wacc, tacc, d.nslots, nwarps, nacc, partials + d.part_off, warp, lane);
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

size_t reg_smem(int k, int nb, int nwarps, int nslots, int nops, int nsegs, bool tiles, bool thread_acc,
                int acc_shift) {
  const size_t tacc = thread_acc ? sizeof(double2) * ((size_t(nslots) * (nwarps * 32 >> acc_shift) + 1) / 2) : 0;
  return sizeof(double2) * (size_t(nwarps) * nslots + (tiles ? (size_t(nb) << k) : 0)) + sizeof(SegDesc) * nsegs +
         sizeof(RegOp) * nops + tacc;
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
