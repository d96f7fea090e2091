// Granular neighbour-list build on the device:
// neighborhood.py:60-101.  One CTA per source node i:
//   finish_ij = (l_i + s_i) + t_ij
//   early     = maximum(e_j - finish_ij, 0)                       (NaN-propagating)
//   late      = isinf(l_j) ? 0 : nan_to_num(maximum(finish_ij - l_j, 0))
//   eta_ij    = c_ij + Gamma * (alpha * early + beta * late)
//   allowed   = !((e_i + s_i) + t_ij > l_j) && j >= n_depots && j != i
// rows sorted ascending by (eta, j) -- np.lexsort((cand, eta)) -- first theta kept.
// Selection: candidates stream through a shared-memory bitonic sorter in chunks;
// the first theta (key, id) pairs of each sorted chunk are carried into the next,
// so any N works with a fixed 4096-slot buffer.  Keys are the order-preserving
// uint64 image of eta (+0.0 folded so -0 == +0; every NaN maps to the top, equal).
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstdint>

#include "../../include/mdr_sm100.h"
#include "mdr_kernels.cuh"

namespace {

constexpr int NB_SLOTS = 4096;
constexpr int NB_THREADS = 512;
constexpr unsigned long long NB_NONE = ~0ull;

__device__ __forceinline__ double np_maximum0(double x) {  // np.maximum(x, 0.0)
  return (x != x) ? x : (x > 0.0 ? x : 0.0);
}

__device__ __forceinline__ unsigned long long eta_key(double eta) {
  if (eta != eta) return NB_NONE - 1;  // NaN: after every number, before "no candidate"
  unsigned long long u = (unsigned long long)__double_as_longlong(eta + 0.0);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ bool nb_less(unsigned long long ka, int ia, unsigned long long kb, int ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(NB_THREADS) k_neighbors(int n, int nd, const double *__restrict__ dist,
                                                          const double *__restrict__ time,
                                                          const double *__restrict__ e, const double *__restrict__ l,
                                                          const double *__restrict__ s, double gamma, double alpha,
                                                          double beta, int theta, int32_t *__restrict__ lists,
                                                          uint8_t *__restrict__ mask) {
  __shared__ unsigned long long sk[NB_SLOTS];
  __shared__ int si[NB_SLOTS];
  const int i = blockIdx.x;
  const double li = l[i], si_ = s[i], ei = e[i];
  const double *crow = dist + (size_t)i * n, *trow = time + (size_t)i * n;
  for (int q = threadIdx.x; q < theta; q += blockDim.x) { sk[q] = NB_NONE; si[q] = 0x7fffffff; }
  const int chunk = NB_SLOTS - theta;
  for (int c0 = nd; c0 < n; c0 += chunk) {
    for (int q = threadIdx.x; q < chunk; q += blockDim.x) {
      const int j = c0 + q;
      unsigned long long key = NB_NONE;
      int id = 0x7fffffff;
      if (j < n && j != i) {
        const double t = trow[j], lj = l[j];
        if (!(((ei + si_) + t) > lj)) {
          const double fin = (li + si_) + t;
          const double early = np_maximum0(e[j] - fin);
          double late = 0.0;
          if (!isinf(lj)) {
            late = np_maximum0(fin - lj);
            if (late != late) late = 0.0;
            else if (isinf(late)) late = late > 0 ? DBL_MAX : -DBL_MAX;
          }
          key = eta_key(crow[j] + gamma * (alpha * early + beta * late));
          id = j;
        }
      }
      sk[theta + q] = key;
      si[theta + q] = id;
    }
    __syncthreads();
    // bitonic sort of NB_SLOTS (key, id) pairs, ascending
    for (int k = 2; k <= NB_SLOTS; k <<= 1) {
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        for (int t = threadIdx.x; t < NB_SLOTS / 2; t += blockDim.x) {
          const int a = 2 * t - (t & (jj - 1)), b = a + jj;
          const bool up = (a & k) == 0;
          const unsigned long long ka = sk[a], kb = sk[b];
          const int ia = si[a], ib = si[b];
          if (nb_less(kb, ib, ka, ia) == up) {
            sk[a] = kb; sk[b] = ka;
            si[a] = ib; si[b] = ia;
          }
        }
        __syncthreads();
      }
    }
  }
  for (int q = threadIdx.x; q < theta; q += blockDim.x)
    lists[(size_t)i * theta + q] = sk[q] == NB_NONE ? -1 : si[q];
  if (mask) {
    uint8_t *mrow = mask + (size_t)i * n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) mrow[j] = 0;
    __syncthreads();
    for (int q = threadIdx.x; q < theta; q += blockDim.x)
      if (sk[q] != NB_NONE) mrow[si[q]] = 1;
  }
}

}  // namespace

extern "C" int mdr_neighbor_build(int32_t device, int32_t n, int32_t n_depots, const double *dist, const double *time,
                                  const double *tw_early, const double *tw_late, const double *service, double gamma,
                                  double alpha, double beta, int32_t theta, int32_t *lists, uint8_t *mask,
                                  float *kernel_ms) {
  if (n < 1 || n_depots < 0 || n_depots > n || theta < 1 || theta > NB_SLOTS / 2 || !dist || !tw_early ||
      !tw_late || !service || !lists)
    return mdr::mdr_fail(MDR_ERR_ARG, "mdr_neighbor_build: bad argument");
  if (cudaSetDevice(device) != cudaSuccess) return mdr::mdr_fail(MDR_ERR_CUDA, "mdr_neighbor_build: cudaSetDevice");
  const size_t nn = (size_t)n * n;
  const bool alias = time == nullptr || time == dist;
  double *dd = nullptr, *dt = nullptr, *dv = nullptr;
  int32_t *dl = nullptr;
  uint8_t *dm = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = MDR_ERR_CUDA;
  do {
    if (cudaMalloc(&dd, nn * sizeof(double)) != cudaSuccess) break;
    if (!alias && cudaMalloc(&dt, nn * sizeof(double)) != cudaSuccess) break;
    if (cudaMalloc(&dv, 3 * (size_t)n * sizeof(double)) != cudaSuccess) break;
    if (cudaMalloc(&dl, (size_t)n * theta * sizeof(int32_t)) != cudaSuccess) break;
    if (mask && cudaMalloc(&dm, nn) != cudaSuccess) break;
    if (cudaMemcpy(dd, dist, nn * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) break;
    if (!alias && cudaMemcpy(dt, time, nn * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) break;
    if (cudaMemcpy(dv, tw_early, n * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(dv + n, tw_late, n * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(dv + 2 * (size_t)n, service, n * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      break;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) break;
    cudaEventRecord(e0);
    k_neighbors<<<n, NB_THREADS>>>(n, n_depots, dd, alias ? dd : dt, dv, dv + n, dv + 2 * (size_t)n, gamma, alpha,
                                   beta, theta, dl, dm);
    cudaEventRecord(e1);
    if (cudaGetLastError() != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess) break;
    if (kernel_ms) cudaEventElapsedTime(kernel_ms, e0, e1);
    if (cudaMemcpy(lists, dl, (size_t)n * theta * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess) break;
    if (mask && cudaMemcpy(mask, dm, nn, cudaMemcpyDeviceToHost) != cudaSuccess) break;
    rc = MDR_OK;
  } while (0);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(dd);
  cudaFree(dt);
  cudaFree(dv);
  cudaFree(dl);
  cudaFree(dm);
  return rc == MDR_OK ? rc : mdr::mdr_fail(rc, "mdr_neighbor_build: CUDA error");
}
