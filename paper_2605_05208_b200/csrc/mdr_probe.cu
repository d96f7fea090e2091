// Diagnostic: L2 read bandwidth of this device (the on-chip roofline
// denominator bench.py reports next to the HBM one; the evaluation kernels'
// working set -- distance rows, route tables -- is L2-resident).
#include <cuda_runtime.h>

#include "../../include/mdr_sm100.h"

namespace {

__global__ void __launch_bounds__(512) k_l2_read(const uint4 *__restrict__ buf, size_t n16, int iters,
                                                 unsigned *sink) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; it++)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(buf + i));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x9e3779b9u) *sink = acc;  // keeps the loads live
}

// 8 independent dmul+dadd chains per thread (no FMA: built with -fmad=false,
// the same arithmetic the evaluators issue); 2 fp64 ops per step per chain.
__global__ void __launch_bounds__(256) k_fp64(double seed, int iters, double *sink) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; j++) x[j] = seed + threadIdx.x + j;
  for (int it = 0; it < iters; it++)
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = x[j] * 0.9999999 + 1e-7;
  double a = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) a += x[j];
  if (a == 1234.5) *sink = a;
}

}  // namespace

extern "C" int mdr_probe_l2_gbs(int32_t device, int64_t bytes, int32_t iters, double *gbs) {
  if (!gbs || bytes < (1 << 20) || iters < 1) return 1;
  if (cudaSetDevice(device) != cudaSuccess) return 4;
  uint4 *buf = nullptr;
  unsigned *sink = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = 4, sms = 148;
  size_t n16 = (size_t)bytes / 16;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&buf, n16 * 16) == cudaSuccess && cudaMalloc(&sink, 4) == cudaSuccess &&
      cudaMemset(buf, 1, n16 * 16) == cudaSuccess && cudaEventCreate(&e0) == cudaSuccess &&
      cudaEventCreate(&e1) == cudaSuccess) {
    k_l2_read<<<sms * 4, 512>>>(buf, n16, 2, sink);  // warm L2
    cudaEventRecord(e0);
    k_l2_read<<<sms * 4, 512>>>(buf, n16, iters, sink);
    cudaEventRecord(e1);
    float ms = 0;
    if (cudaEventSynchronize(e1) == cudaSuccess && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess &&
        ms > 0) {
      *gbs = (double)n16 * 16 * iters / (ms * 1e-3) / 1e9;
      rc = 0;
    }
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(sink);
  return rc;
}

extern "C" int mdr_probe_fp64_gops(int32_t device, int32_t iters, double *gops) {
  if (!gops || iters < 1) return 1;
  if (cudaSetDevice(device) != cudaSuccess) return 4;
  double *sink = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = 4, sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = sms * 8, threads = 256;
  if (cudaMalloc(&sink, 8) == cudaSuccess && cudaEventCreate(&e0) == cudaSuccess &&
      cudaEventCreate(&e1) == cudaSuccess) {
    k_fp64<<<blocks, threads>>>(1.0, 64, sink);
    cudaEventRecord(e0);
    k_fp64<<<blocks, threads>>>(1.0, iters, sink);
    cudaEventRecord(e1);
    float ms = 0;
    if (cudaEventSynchronize(e1) == cudaSuccess && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess &&
        ms > 0) {
      *gops = (double)blocks * threads * iters * 16.0 / (ms * 1e-3) / 1e9;
      rc = 0;
    }
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(sink);
  return rc;
}
