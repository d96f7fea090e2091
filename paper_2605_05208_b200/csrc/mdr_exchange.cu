// mdr_exchange.cu -- the route exchange of DCREX on the device (SURVEY.md 8(f)
// row 3; reference genetic.py:343-446): one CTA per offspring builds it from
// the population's members, so a lock-step generation's B exchanges run
// together instead of one after the other on the host.
//
// Per offspring (main parent, donor order and the MT19937 state after those
// draws come from the host, exactly as `rng.randrange` / `rng.shuffle` left
// them): the offspring starts as the main parent; for every donor, repeatedly
// score every (main-origin offspring route oi, unused non-empty donor route dj)
// pair (score_route_pair, genetic.py:316-330: new edges of dj absent from the
// main parent, customers of oi dj misses, dj's customers already in other
// main-origin routes, dj's customers clashing with introduced ones), take the
// five smallest (score, oi, dj), draw one with CPython's choice
// (_randbelow_with_getrandbits on the continued MT19937 stream), stop the donor
// when sigma would reach sigma_max, else exchange and stop everything once
// sigma reaches sigma_min.  Then _remove_redundant (genetic.py:424-446): of a
// duplicated customer the donor copy is kept first, then the copy whose
// removal saves least (first on ties), and the unrouted customers are listed.
// Integer bookkeeping is exact; the removal savings use the reference's fp64
// expression (-fmad=false), so the offspring equal the host route_exchange.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/mdr_sm100.h"
#include "mdr_kernels.cuh"

namespace mdr {

constexpr int XC_THREADS = 128;

// CPython genrand_uint32 (Modules/_randommodule.c)
__device__ uint32_t xc_mt_next(uint32_t *mt, uint32_t &idx) {
  const int N = 624, M = 397;
  const uint32_t A = 0x9908b0dfU, UP = 0x80000000U, LO = 0x7fffffffU;
  uint32_t y;
  if (idx >= (uint32_t)N) {
    int kk;
    for (kk = 0; kk < N - M; kk++) {
      y = (mt[kk] & UP) | (mt[kk + 1] & LO);
      mt[kk] = mt[kk + M] ^ (y >> 1) ^ ((y & 1U) ? A : 0U);
    }
    for (; kk < N - 1; kk++) {
      y = (mt[kk] & UP) | (mt[kk + 1] & LO);
      mt[kk] = mt[kk + (M - N)] ^ (y >> 1) ^ ((y & 1U) ? A : 0U);
    }
    y = (mt[N - 1] & UP) | (mt[0] & LO);
    mt[N - 1] = mt[M - 1] ^ (y >> 1) ^ ((y & 1U) ? A : 0U);
    idx = 0;
  }
  y = mt[idx++];
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680U;
  y ^= (y << 15) & 0xefc60000U;
  y ^= (y >> 18);
  return y;
}

// Random._randbelow_with_getrandbits(n), n >= 1 (n <= 2^31)
__device__ int xc_randbelow(uint32_t *mt, uint32_t &idx, int n) {
  const int k = 32 - __clz(n);  // n.bit_length()
  uint32_t r = xc_mt_next(mt, idx) >> (32 - k);
  while (r >= (uint32_t)n) r = xc_mt_next(mt, idx) >> (32 - k);
  return (int)r;
}

__device__ __forceinline__ bool xc_bit(const unsigned *bm, int x) { return (bm[x >> 5] >> (x & 31)) & 1u; }

// edge (a, b) of a route is in the main parent's edge set: b is a's neighbour in main
// (every route edge has a customer end; prv/nxt of a customer in its main route, -1 none)
__device__ __forceinline__ bool xc_in_main(const DevInst &I, const int *prv, const int *nxt, int a, int b) {
  if (a >= I.ND) return prv[a] == b || nxt[a] == b;
  return prv[b] == a || nxt[b] == a;
}

__global__ void __launch_bounds__(XC_THREADS) k_exchange(DevInst I, XcPop X, XcJob Jb, XcOut O, int M, int *g_prv,
                                                         int *g_nxt, int *g_owner, unsigned *g_bits, int *g_cnt,
                                                         long long *g_key, int cnt_cap) {
  const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int N = I.N, words = (N + 31) / 32;
  __shared__ uint32_t s_mt[625];
  __shared__ int s_nref, s_err, s_done, s_nin, s_nout, s_pick, s_npairs, s_ro;
  __shared__ double s_sigma;
  __shared__ long long s_best[XC_THREADS / 32];
  __shared__ long long s_top[5];
  int *prv = g_prv + (size_t)j * N, *nxt = g_nxt + (size_t)j * N, *owner = g_owner + (size_t)j * N;
  unsigned *MC = g_bits + (size_t)j * 3 * words, *INTRO = MC + words, *USED = INTRO + words;
  int *cnt = g_cnt + (size_t)j * cnt_cap;  // inter [nout][nin], then per-dj new edges / in_mc / n_c
  long long *key = g_key + (size_t)j * cnt_cap;
  int *refs = O.refs + (size_t)j * O.Jcap, *orig = O.orig + (size_t)j * O.Jcap;
  for (int i = tid; i < 625; i += XC_THREADS) s_mt[i] = Jb.mt[(size_t)j * 625 + i];
  const int mainm = Jb.main[j];
  for (int v = tid; v < N; v += XC_THREADS) { prv[v] = -1; nxt[v] = -1; owner[v] = -1; }
  for (int w = tid; w < 3 * words; w += XC_THREADS) MC[w] = 0u;
  if (tid == 0) { s_err = 0; s_done = 0; s_sigma = 0.0; }
  __syncthreads();
  const double sig_min = Jb.sig[2 * j], sig_max = Jb.sig[2 * j + 1];
  // the offspring starts as the main parent (all its routes, in order)
  {
    const int r0 = X.mroute[mainm], r1 = X.mroute[mainm + 1];
    if (r1 - r0 > O.Jcap) s_err = MDR_ERR_CAPACITY;
    for (int r = r0 + tid; r < r1; r += XC_THREADS) {
      refs[r - r0] = r;
      orig[r - r0] = 1;
      const int c0 = X.coff[r], c1 = X.coff[r + 1];
      for (int p = c0; p < c1; p++) {
        const int c = X.cust[p];
        prv[c] = p == c0 ? X.dep[r] : X.cust[p - 1];
        nxt[c] = p + 1 < c1 ? X.cust[p + 1] : (I.open ? -1 : X.arr[r]);
        owner[c] = r - r0;
        atomicOr(&MC[c >> 5], 1u << (c & 31));
      }
    }
    if (tid == 0) s_nref = r1 - r0;
  }
  __syncthreads();
  if (s_err) { if (tid == 0) O.status[j] = s_err; return; }
  uint32_t mtidx = 0;
  if (tid == 0) mtidx = s_mt[624];
  for (int di = 0; di < M - 1 && !s_done; di++) {
    const int dm = Jb.donors[(size_t)j * (M - 1) + di];
    const int d0 = X.mroute[dm], nd = X.mroute[dm + 1] - d0;
    for (int w = tid; w < (nd + 31) / 32; w += XC_THREADS) USED[w] = 0u;
    __syncthreads();
    for (;;) {
      // outs: main-origin offspring routes (owner indexes are offspring route slots);
      // ins: unused non-empty donor routes
      if (tid == 0) {
        int no = 0, ni = 0;
        for (int o = 0; o < s_nref; o++) no += orig[o];
        for (int d = 0; d < nd; d++) ni += !xc_bit(USED, d) && X.coff[d0 + d + 1] > X.coff[d0 + d];
        s_nout = no; s_nin = ni;
        s_npairs = no * ni;
      }
      __syncthreads();
      const int nref = s_nref, npairs = s_npairs;
      if (npairs == 0) break;
      if ((long long)nref * nd + 3 * nd > cnt_cap) { if (tid == 0) s_err = MDR_ERR_CAPACITY; break; }
      // per (offspring slot o, donor route d): intersections; per d: new edges, in MC, introduced
      int *inter = cnt, *e_new = cnt + nref * nd, *in_mc = e_new + nd, *n_c = in_mc + nd;
      for (int i = tid; i < nref * nd + 3 * nd; i += XC_THREADS) cnt[i] = 0;
      __syncthreads();
      for (int d = wid; d < nd; d += XC_THREADS / 32) {
        const int r = d0 + d, c0 = X.coff[r], c1 = X.coff[r + 1];
        if (c1 == c0 || xc_bit(USED, d)) continue;
        int en = 0, im = 0, ic = 0;
        const bool single_loop = !I.open && c1 - c0 == 1 && X.dep[r] == X.arr[r];
        for (int p = c0 + lane; p < c1; p += 32) {
          const int c = X.cust[p];
          const int a = p == c0 ? X.dep[r] : X.cust[p - 1];
          en += !xc_in_main(I, prv, nxt, a, c);  // edge (previous node, c)
          if (p + 1 == c1 && !I.open && !single_loop) en += !xc_in_main(I, prv, nxt, c, X.arr[r]);
          im += xc_bit(MC, c);
          ic += xc_bit(INTRO, c);
          const int o = owner[c];
          if (o >= 0 && orig[o]) atomicAdd(&inter[o * nd + d], 1);
        }
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
          en += __shfl_xor_sync(0xffffffffu, en, s);
          im += __shfl_xor_sync(0xffffffffu, im, s);
          ic += __shfl_xor_sync(0xffffffffu, ic, s);
        }
        if (lane == 0) { e_new[d] = en; in_mc[d] = im; n_c[d] = ic; }
      }
      __syncthreads();
      // keys of every admissible pair: (score, oi, dj) with oi the offspring slot
      for (int i = tid; i < nref * nd; i += XC_THREADS) {
        const int o = i / nd, d = i - o * nd, r = d0 + d;
        long long k = 0x7fffffffffffffffll;
        if (orig[o] && !xc_bit(USED, d) && X.coff[r + 1] > X.coff[r]) {
          const int ro = refs[o], k_out = X.coff[ro + 1] - X.coff[ro];
          const int it = inter[i], missing = k_out - it, dup = in_mc[d] - it;
          const int score = -(e_new[d] - missing - dup - 10 * n_c[d]);
          k = ((long long)(score + (1 << 29)) << 32) | ((long long)o << 16) | d;
        }
        key[i] = k;
      }
      __syncthreads();
      // the five smallest keys, ascending (sorted(pairs)[:5])
      const int ntop = npairs < 5 ? npairs : 5;
      for (int t = 0; t < ntop; t++) {
        long long best = 0x7fffffffffffffffll;
        for (int i = tid; i < nref * nd; i += XC_THREADS) {
          const long long k = key[i];
          bool taken = false;
          for (int u = 0; u < t; u++) taken |= s_top[u] == k;
          if (!taken && k < best) best = k;
        }
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
          const long long o2 = __shfl_xor_sync(0xffffffffu, best, s);
          if (o2 < best) best = o2;
        }
        if (lane == 0) s_best[wid] = best;
        __syncthreads();
        if (tid == 0) {
          long long b2 = s_best[0];
          for (int w = 1; w < XC_THREADS / 32; w++) b2 = s_best[w] < b2 ? s_best[w] : b2;
          s_top[t] = b2;
        }
        __syncthreads();
      }
      if (tid == 0) {
        const long long k = s_top[xc_randbelow(s_mt, mtidx, ntop)];  // rng.choice(pairs[:5])
        const int o = (int)((k >> 16) & 0xffff), d = (int)(k & 0xffff);
        const int ro = refs[o], k_out = X.coff[ro + 1] - X.coff[ro];
        const int it = inter[o * nd + d], missing = k_out - it, dup = in_mc[d] - it;
        const int ds = e_new[d] + missing + dup;
        s_pick = -1;
        if (!(s_sigma + (double)ds >= sig_max)) {
          s_pick = o;
          s_sigma += (double)ds;
          // the offspring drops slot o (later slots shift down) and appends donor route d
          for (int q = o; q + 1 < s_nref; q++) { refs[q] = refs[q + 1]; orig[q] = orig[q + 1]; }
          refs[s_nref - 1] = d0 + d;
          orig[s_nref - 1] = 0;
          USED[d >> 5] |= 1u << (d & 31);
          if (s_sigma >= sig_min) s_done = 1;
          s_ro = ro;  // the removed member route (its customers leave MC)
        }
      }
      __syncthreads();
      if (s_pick < 0) break;  // this donor would overshoot the window: next donor
      {
        const int o = s_pick, ro = s_ro, rn = refs[s_nref - 1];
        for (int p = X.coff[ro] + tid; p < X.coff[ro + 1]; p += XC_THREADS) {
          const int c = X.cust[p];
          atomicAnd(&MC[c >> 5], ~(1u << (c & 31)));
          owner[c] = -1;
        }
        __syncthreads();
        for (int v = tid; v < N; v += XC_THREADS)
          if (owner[v] > o) owner[v]--;
        for (int p = X.coff[rn] + tid; p < X.coff[rn + 1]; p += XC_THREADS) {
          const int c = X.cust[p];
          atomicOr(&INTRO[c >> 5], 1u << (c & 31));
        }
      }
      __syncthreads();
      if (s_done) break;
    }
    __syncthreads();
    if (s_err) break;
  }
  __syncthreads();
  if (s_err) { if (tid == 0) O.status[j] = s_err; return; }
  // _remove_redundant: slots of the offspring's customers in (route, position) order
  const int nref = s_nref;
  int *keep = O.keep + (size_t)j * O.Ccap;
  if (tid == 0) {
    int tot = 0;
    for (int o = 0; o < nref; o++) tot += X.coff[refs[o] + 1] - X.coff[refs[o]];
    if (tot > O.Ccap) s_err = MDR_ERR_CAPACITY;
    s_npairs = tot;
  }
  __syncthreads();
  if (s_err) { if (tid == 0) O.status[j] = s_err; return; }
  // per customer: its best copy so far as (origin, saving, slot) -- a sequential
  // pass in slot order keeps the reference's min-first tie order
  if (tid == 0) {
    int at = 0;
    for (int v = 0; v < N; v++) owner[v] = -1;  // best slot per customer
    double *bestsave = reinterpret_cast<double *>(key);  // [N] scratch (cnt_cap >= N)
    for (int o = 0; o < nref; o++) {
      const int r = refs[o], c0 = X.coff[r], c1 = X.coff[r + 1];
      for (int p = c0; p < c1; p++, at++) {
        const int c = X.cust[p];
        const int prevn = p == c0 ? X.dep[r] : X.cust[p - 1];
        double save;
        const bool last = p + 1 == c1;
        if (last && I.open) {
          save = I.dist[(size_t)prevn * N + c];
        } else {
          const int nx = last ? X.arr[r] : X.cust[p + 1];
          save = (I.dist[(size_t)prevn * N + c] + I.dist[(size_t)c * N + nx]) - I.dist[(size_t)prevn * N + nx];
        }
        keep[at] = 0;
        const int cur = owner[c];
        if (cur < 0) {
          owner[c] = at;
          prv[c] = orig[o];
          bestsave[c] = save;
        } else if (orig[o] < prv[c] || (orig[o] == prv[c] && save < bestsave[c])) {
          owner[c] = at;
          prv[c] = orig[o];
          bestsave[c] = save;
        }
      }
    }
    for (int v = 0; v < N; v++)
      if (owner[v] >= 0) keep[owner[v]] = 1;
    int nu = 0;
    int *unr = O.unr + (size_t)j * (N - I.ND);
    for (int v = I.ND; v < N; v++)
      if (owner[v] < 0) unr[nu++] = v;
    O.nunr[j] = nu;
    O.nref[j] = nref;
    for (int i = 0; i < 624; i++) Jb.mt[(size_t)j * 625 + i] = s_mt[i];  // the stream after the choices
    Jb.mt[(size_t)j * 625 + 624] = mtidx;
    O.sigma[j] = s_sigma;
    O.status[j] = 0;
  }
}

void launch_exchange(const DevInst &I, const XcPop &X, const XcJob &Jb, const XcOut &O, int B, int M, int *prv,
                     int *nxt, int *owner, unsigned *bits, int *cnt, long long *key, int cnt_cap, cudaStream_t s) {
  if (B > 0) k_exchange<<<B, XC_THREADS, 0, s>>>(I, X, Jb, O, M, prv, nxt, owner, bits, cnt, key, cnt_cap);
}

}  // namespace mdr
