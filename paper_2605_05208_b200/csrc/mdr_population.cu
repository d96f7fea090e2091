// mdr_population.cu -- population management of the generation loop on the
// device: edge-set distances between members and the
// fitness-and-diversity survivor selection.
//
// Reference: population.py:19-24 (solution_distance), 27-34
// (population_distance), 51-67 (biased_fitness), 94-116 (distance matrix and
// survivor_selection).  Edge sets are passed as sorted, de-duplicated int64
// keys a*N+b (a <= b) -- model.py:217-228 route_edges/solution_edges.
//
// Distances: one warp per (new row i, column j) pair; the lanes stride over the
// shorter key array and binary-search the longer one, so a pair costs
// O(min |E| log max |E|) with no shared state; the count is exact, and the
// distance 100 * (1 - inter / max(|Ei|, |Ej|)) is formed with the reference's
// operation order (IEEE division of exactly representable integers).
//
// Survivor selection: one CTA holds the alive set and repeats the reference's
// round: population_distance of every alive member (mean of its five smallest
// distances, summed in ascending order from 0), rank by (cost, birth) and by
// (-diversity, birth) (ranks by counting: births are unique, so the order is
// total), chi = (n - rank_f)/n + xi*(n - rank_d)/n, and drop the member of
// minimal (chi, birth).  Bit-identical to the Python loop; O(n^2) per round
// spread over the CTA instead of a Python O(n^2 log n).
#include <cuda_runtime.h>
#include <cstdint>
#include <cmath>

namespace mdr {

__global__ void k_edge_dist(int n, int row0, const long long *off, const long long *keys, double *dist) {
  const int lane = threadIdx.x & 31;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long rows = n - row0;
  if (w >= rows * n) return;
  const int i = row0 + (int)(w / n), j = (int)(w % n);
  if (i == j) {
    if (lane == 0) dist[(size_t)i * n + j] = 0.0;
    return;
  }
  if (j >= row0 && j > i) return;  // the pair (j, i) of two new rows is done by row j
  const long long ai = off[i], ni = off[i + 1] - ai, aj = off[j], nj = off[j + 1] - aj;
  double d;
  if (ni == 0 && nj == 0) {
    d = 0.0;
  } else {
    const long long *S = ni <= nj ? keys + ai : keys + aj, *Lg = ni <= nj ? keys + aj : keys + ai;
    const long long ns = ni <= nj ? ni : nj, nl = ni <= nj ? nj : ni;
    long long cnt = 0;
    for (long long t = lane; t < ns; t += 32) {
      const long long x = S[t];
      long long lo = 0, hi = nl;
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (Lg[mid] < x) lo = mid + 1;
        else hi = mid;
      }
      cnt += (lo < nl && Lg[lo] == x) ? 1 : 0;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, s);
    d = 100.0 * (1.0 - (double)cnt / (double)nl);
  }
  if (lane == 0) {
    dist[(size_t)i * n + j] = d;
    dist[(size_t)j * n + i] = d;
  }
}

// lexicographic (a, birth) compare, births unique
__device__ __forceinline__ bool lt2(double a, long long ba, double b, long long bb) {
  return a < b || (a == b && ba < bb);
}

__global__ void __launch_bounds__(1024) k_survivors(int n, int mu, double xi, const double *dist, const double *cost,
                                                     const long long *birth, unsigned char *alive, double *div,
                                                     int *removed) {
  __shared__ double s_chi[32];
  __shared__ long long s_b[32];
  __shared__ int s_i[32];
  __shared__ int s_worst;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < n; i += blockDim.x) alive[i] = 1;
  __syncthreads();
  int na = n, nrem = 0;
  while (na > mu) {
    // population_distance of every alive member (population.py:27-34)
    for (int i = tid; i < n; i += blockDim.x) {
      if (!alive[i]) continue;
      double best[5];
      int nb = 0;
      const double *row = dist + (size_t)i * n;
      for (int j = 0; j < n; j++) {
        if (j == i || !alive[j]) continue;
        double x = row[j];
        if (nb < 5) {  // insertion into the ascending list
          int p = nb++;
          while (p > 0 && best[p - 1] > x) { best[p] = best[p - 1]; p--; }
          best[p] = x;
        } else if (x < best[4]) {
          int p = 4;
          while (p > 0 && best[p - 1] > x) { best[p] = best[p - 1]; p--; }
          best[p] = x;
        }
      }
      double s = 0.0;
      for (int q = 0; q < nb; q++) s = s + best[q];
      div[i] = nb ? s / (double)nb : 0.0;
    }
    __syncthreads();
    // biased fitness (population.py:51-67) and the argmin over (chi, birth)
    double bc = INFINITY;
    long long bb = 0x7fffffffffffffffll;
    int bi = -1;
    const double nd = (double)na;
    for (int i = tid; i < n; i += blockDim.x) {
      if (!alive[i]) continue;
      int rf = 0, rd = 0;
      const double ci = cost[i], di = -div[i];
      const long long bi_ = birth[i];
      for (int j = 0; j < n; j++) {
        if (!alive[j] || j == i) continue;
        rf += lt2(cost[j], birth[j], ci, bi_);
        rd += lt2(-div[j], birth[j], di, bi_);
      }
      const double chi = (double)(na - rf) / nd + (xi * (double)(na - rd)) / nd;
      if (bi < 0 || lt2(chi, bi_, bc, bb)) { bc = chi; bb = bi_; bi = i; }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const double oc = __shfl_xor_sync(0xffffffffu, bc, s);
      const long long ob = __shfl_xor_sync(0xffffffffu, bb, s);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, s);
      if (oi >= 0 && (bi < 0 || lt2(oc, ob, bc, bb))) { bc = oc; bb = ob; bi = oi; }
    }
    if (lane == 0) { s_chi[wid] = bc; s_b[wid] = bb; s_i[wid] = bi; }
    __syncthreads();
    if (wid == 0) {
      bc = lane < nw ? s_chi[lane] : INFINITY;
      bb = lane < nw ? s_b[lane] : 0x7fffffffffffffffll;
      bi = lane < nw ? s_i[lane] : -1;
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        const double oc = __shfl_xor_sync(0xffffffffu, bc, s);
        const long long ob = __shfl_xor_sync(0xffffffffu, bb, s);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, s);
        if (oi >= 0 && (bi < 0 || lt2(oc, ob, bc, bb))) { bc = oc; bb = ob; bi = oi; }
      }
      if (lane == 0) {
        s_worst = bi;
        alive[bi] = 0;
        removed[nrem] = bi;
      }
    }
    __syncthreads();
    nrem++;
    na--;
  }
}

void launch_edge_dist(int n, int row0, const long long *off, const long long *keys, double *dist, cudaStream_t s) {
  const long long warps = (long long)(n - row0) * n;
  if (warps <= 0) return;
  const long long blocks = (warps * 32 + 255) / 256;
  k_edge_dist<<<(unsigned)blocks, 256, 0, s>>>(n, row0, off, keys, dist);
}

void launch_survivors(int n, int mu, double xi, const double *dist, const double *cost, const long long *birth,
                      unsigned char *alive, double *div, int *removed, cudaStream_t s) {
  k_survivors<<<1, 1024, 0, s>>>(n, mu, xi, dist, cost, birth, alive, div, removed);
}

}  // namespace mdr

#include "../../include/mdr_sm100.h"
#include "mdr_kernels.cuh"

extern "C" int mdr_population_select(int32_t device, int32_t n, int32_t row0, const int64_t *edge_off,
                                     const int64_t *edge_keys, double *dist, int32_t mu, double xi,
                                     const double *cost, const int64_t *birth, int32_t *removed) {
  if (n < 0 || row0 < 0 || row0 > n || mu < 0 || !edge_off || !dist || (n > mu && (!cost || !birth || !removed)))
    return mdr::mdr_fail(MDR_ERR_ARG, "mdr_population_select: bad argument");
  if (n == 0) return MDR_OK;
  if (cudaSetDevice(device) != cudaSuccess) return mdr::mdr_fail(MDR_ERR_CUDA, "mdr_population_select: cudaSetDevice");
  const size_t nn = (size_t)n * n;
  const long long nk = edge_off[n];
  for (int i = 0; i < n; i++)
    if (edge_off[i + 1] < edge_off[i]) return mdr::mdr_fail(MDR_ERR_ARG, "mdr_population_select: edge_off must be non-decreasing");
  long long *d_off = nullptr, *d_keys = nullptr, *d_birth = nullptr;
  double *d_dist = nullptr, *d_cost = nullptr, *d_div = nullptr;
  unsigned char *d_alive = nullptr;
  int *d_rem = nullptr;
  int rc = MDR_ERR_CUDA;
  const int nrem = n > mu ? n - mu : 0;
  do {
    if (cudaMallocAsync(&d_off, sizeof(long long) * (n + 1), 0) != cudaSuccess) break;
    if (cudaMallocAsync(&d_keys, sizeof(long long) * (nk > 0 ? nk : 1), 0) != cudaSuccess) break;
    if (cudaMallocAsync(&d_dist, sizeof(double) * nn, 0) != cudaSuccess) break;
    if (cudaMemcpy(d_off, edge_off, sizeof(long long) * (n + 1), cudaMemcpyHostToDevice) != cudaSuccess) break;
    if (nk > 0 && cudaMemcpy(d_keys, edge_keys, sizeof(long long) * nk, cudaMemcpyHostToDevice) != cudaSuccess) break;
    if (cudaMemcpy(d_dist, dist, sizeof(double) * nn, cudaMemcpyHostToDevice) != cudaSuccess) break;
    mdr::launch_edge_dist(n, row0, d_off, d_keys, d_dist, 0);
    if (cudaGetLastError() != cudaSuccess) break;
    if (nrem) {
      if (cudaMallocAsync(&d_cost, sizeof(double) * n, 0) != cudaSuccess) break;
      if (cudaMallocAsync(&d_birth, sizeof(long long) * n, 0) != cudaSuccess) break;
      if (cudaMallocAsync(&d_div, sizeof(double) * n, 0) != cudaSuccess) break;
      if (cudaMallocAsync(&d_alive, n, 0) != cudaSuccess) break;
      if (cudaMallocAsync(&d_rem, sizeof(int) * nrem, 0) != cudaSuccess) break;
      if (cudaMemcpy(d_cost, cost, sizeof(double) * n, cudaMemcpyHostToDevice) != cudaSuccess) break;
      if (cudaMemcpy(d_birth, birth, sizeof(long long) * n, cudaMemcpyHostToDevice) != cudaSuccess) break;
      mdr::launch_survivors(n, mu, xi, d_dist, d_cost, d_birth, d_alive, d_div, d_rem, 0);
      if (cudaGetLastError() != cudaSuccess) break;
      if (cudaMemcpy(removed, d_rem, sizeof(int) * nrem, cudaMemcpyDeviceToHost) != cudaSuccess) break;
    }
    if (cudaMemcpy(dist, d_dist, sizeof(double) * nn, cudaMemcpyDeviceToHost) != cudaSuccess) break;
    rc = MDR_OK;
  } while (0);
  if (d_off) cudaFreeAsync(d_off, 0);
  if (d_keys) cudaFreeAsync(d_keys, 0);
  if (d_dist) cudaFreeAsync(d_dist, 0);
  if (d_cost) cudaFreeAsync(d_cost, 0);
  if (d_birth) cudaFreeAsync(d_birth, 0);
  if (d_div) cudaFreeAsync(d_div, 0);
  if (d_alive) cudaFreeAsync(d_alive, 0);
  if (d_rem) cudaFreeAsync(d_rem, 0);
  return rc == MDR_OK ? rc : mdr::mdr_fail(rc, "mdr_population_select: CUDA error");
}
