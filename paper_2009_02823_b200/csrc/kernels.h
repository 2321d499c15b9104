// Host-callable launchers for the tile-pass kernels (kernels.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace svgb {

size_t fwd_smem(int k, int b);
size_t obs_smem(int k, int b, int nterms);
size_t rev_smem(int k, int b, int nslots);
size_t prod_smem(int k, int b);
cudaError_t prepare_kernels(size_t max_smem);
int occupancy(int which /*0 fwd, 1 obs, 2 rev, 3 product term*/, size_t smem);

void launch_fwd(const PassDesc& d, int grid, size_t smem, cudaStream_t s, double2* psi,
                const DevOp* ops, const double2* coef);
void launch_obs(const PassDesc& d, int grid, size_t smem, cudaStream_t s, const double2* psi, const double2* src,
                double2* lam, const DevTerm* terms, double2* partials);
void launch_prod(const PassDesc& d, const ProdFactors& f, int grid, size_t smem, cudaStream_t s, const double2* src,
                 double2* dst, const double2* psi, double2* lam, double2 scalar, double2* partials);
void launch_obs_direct(const PassDesc& d, int grid, cudaStream_t s, const double2* psi, const double2* src,
                       double2* lam, const DevTerm* terms, double2* partials);
// qubit swap of a sharded state (virtual shards in one allocation): for every
// shard pair differing in rank bit `gbit`, exchange lower's amplitudes with
// local bit `lpos` = 1 and upper's with local bit `lpos` = 0.
void launch_swap_virtual(double2* state, int nloc, int nshards, int gbit, int lpos, cudaStream_t s);
// gather / scatter the half of a shard whose local bit `lpos` equals `val` (NCCL exchange staging)
void launch_half_pack(const double2* shard, double2* packed, int nloc, int lpos, int val, cudaStream_t s);
void launch_half_unpack(const double2* packed, double2* shard, int nloc, int lpos, int val, cudaStream_t s);
void launch_rev(const PassDesc& d, int grid, size_t smem, cudaStream_t s, double2* phi, double2* lam,
                const DevOp* ops, const double2* coef, double2* partials);
void launch_finalize(const double2* partials, const SumSpec* specs, int count, double2* out,
                     cudaStream_t s);
void launch_set_basis(double2* psi, uint64_t idx, cudaStream_t s);

// register-tile passes (kernels_reg.cu)
size_t reg_smem(int k, int nb, int nwarps, int nslots, int nops, int nsegs, bool tiles, bool thread_acc,
                int acc_shift);
cudaError_t prepare_reg_kernels(size_t max_smem);
int reg_occupancy(int nb, int R, int threads, size_t smem);
int reg_max_threads(int R);
void launch_pass_reg(int nb, int R, const PassDesc& d, int grid, int threads, size_t smem, cudaStream_t s, double2* b0,
                     double2* b1, const SegDesc* segs, const RegOp* rops, const DevOp* ops, const double2* coef,
                     double2* partials);

}  // namespace svgb
