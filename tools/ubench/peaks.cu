// Micro-benchmarks for the roofline denominators this path needs beyond
// MEASURED_PEAKS.json: FP64 FMA throughput, and read+write bandwidth of a
// double2 stream whose working set fits L2 (the L2-blocked pass regime) vs HBM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, double a, double b, int iters) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void rw_kernel(double2* p, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = p[i];
      v.x = v.x * 0.999999 + 1e-300;
      p[i] = v;
    }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps = 4; warps <= 32; warps *= 2) {
    const int iters = 4096, thr = warps * 32, blocks = sms;
    dfma_kernel<<<blocks, thr>>>(out, 0.9999, 1e-3, 16);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, thr>>>(out, 0.9999, 1e-3, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = double(blocks) * thr * iters * 16 * 8;
    printf("{\"dfma_warps_per_sm\": %d, \"dfma_per_s\": %.4e, \"fp64_tflops\": %.2f}\n", warps, fmas / (ms * 1e-3),
           2 * fmas / (ms * 1e-3) / 1e12);
  }
  for (size_t mb : {16, 32, 48, 64, 96, 128, 4096}) {
    const size_t n = mb * (1 << 20) / 16;
    double2* p;
    cudaMalloc(&p, n * 16);
    cudaMemset(p, 0, n * 16);
    const int reps = mb >= 1024 ? 2 : 20;
    rw_kernel<<<sms * 8, 256>>>(p, n, 1);
    cudaEventRecord(e0);
    rw_kernel<<<sms * 8, 256>>>(p, n, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"rw_working_set_mb\": %zu, \"l2_bytes\": %d, \"gbs\": %.1f}\n", mb, l2, 2.0 * n * 16 * reps / (ms * 1e-3) / 1e9);
    cudaFree(p);
  }
  return 0;
}
