// Repair insertion on the device: genetic.repair_insert
// (genetic.py:174-244) for FBI/IBI/FRI/IRI, batched over the individuals of a
// population -- one CTA per individual, the whole insertion loop on the device.
//
// The reference re-scans every (pending customer x slot) after each insertion.
// Only the inserted-into route's slots change, so this keeps, per (pending
// customer q, route r), the route-local scan summary (m1 = first minimal cost,
// its position, m2 = second-smallest cost of the multiset) and re-scans only
// the touched route's column.  Folding the per-route summaries in route order,
//   m1 <  C1: C2 = min(C1, m2), C1 = m1, slot = (r, pos1)
//   m1 >= C1: C2 = min(C2, m1)
// gives exactly _best_slot's (slot, c1, c2) over the full scan (strict '<'
// keeps the first minimum; c2 is the second-smallest value, multiplicity kept).
//
// Arithmetic follows the scalar evaluation.concat (evaluation.py:74-94) with
// Python's max/min (first argument unless the second is strictly larger /
// smaller); _RouteEval's suffixes are RIGHT folds (genetic.py:87-90).
#include <cuda_runtime.h>

#include <math_constants.h>

#include "../../include/mdr_sm100.h"
#include "mdr_kernels.cuh"

namespace mdr {

struct RAt {
  double dist, load, T, E, L, TW;
};

__device__ __forceinline__ double py_max(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double py_min(double a, double b) { return b < a ? b : a; }

__device__ __forceinline__ RAt r_single(const DevInst &I, int v) {
  const double4 nd = I.node[v];
  RAt a;
  a.dist = 0.0; a.load = nd.x; a.T = nd.y; a.E = nd.z; a.L = nd.w; a.TW = 0.0;
  return a;
}

// concat(a, b) with a.last = x, b.first = y (both non-empty)
__device__ __forceinline__ RAt r_cat(const DevInst &I, const RAt &a, int x, const RAt &b, int y) {
  const size_t lk = (size_t)x * I.N + y;
  const double c = I.dist[lk], t = I.talias ? c : I.time[lk];
  const double delta = (a.T - a.TW) + t;
  const double wait = py_max((b.E - delta) - a.L, 0.0);
  const double warp = py_max((a.E + delta) - b.L, 0.0);
  RAt o;
  o.dist = (a.dist + c) + b.dist;
  o.load = a.load + b.load;
  o.T = ((a.T + b.T) + t) + wait;
  o.E = py_max(b.E - delta, a.E) - wait;
  o.L = py_min(b.L - delta, a.L) + warp;
  o.TW = (a.TW + b.TW) + warp;
  return o;
}

// _route_cost_terms (genetic.py:100-106)
__device__ __forceinline__ void r_terms(const DevInst &I, const RAt &a, double o[4]) {
  o[0] = a.dist;
  o[1] = I.win ? I.gamma * a.TW : 0.0;
  o[2] = (I.theta * py_max(a.load - I.Q, 0.0)) / I.Q;
  o[3] = I.d_on ? (I.theta * py_max(a.T - I.Dmax, 0.0)) / I.Dmax : 0.0;
}

// _attr_feasible (genetic.py:109-116)
__device__ __forceinline__ bool r_feasible(const DevInst &I, const RAt &a) {
  if (a.load > I.Q + 1e-9) return false;
  if (I.d_on && a.T > I.Dmax + 1e-9) return false;
  if (I.win && a.TW > 1e-9) return false;
  return true;
}

struct RepView {
  int *seq;         // [J][Kp] this individual's rows
  int4 *rm;         // [J]
  RAt *pre, *suf;   // [J][Kp]
  double *c1, *c2;  // [Pcap][J]
  int *p1;          // [Pcap][J]
  double *fC1, *fC2;  // [Pcap] per-customer fold over all routes
  int *fR1, *fP1, *fR2;
  int Kp, J, K, Pcap;
};

// fold the per-route summaries of customer q in route order (see the header)
__device__ void r_fold(const RepView &V, int q, int m) {
  double C1 = CUDART_INF, C2 = CUDART_INF;
  int R1 = -1, P1 = -1, R2 = -1;
  const double *c1 = V.c1 + (size_t)q * V.J, *c2 = V.c2 + (size_t)q * V.J;
  const int *p1 = V.p1 + (size_t)q * V.J;
  for (int r = 0; r < m; r++) {
    const double a1 = c1[r];
    if (a1 < C1) {
      const double a2 = c2[r];
      if (a2 < C1) { C2 = a2; R2 = r; }
      else { C2 = C1; R2 = R1; }
      C1 = a1; R1 = r; P1 = p1[r];
    } else if (a1 < C2) {
      C2 = a1; R2 = r;
    }
  }
  V.fC1[q] = C1; V.fC2[q] = C2; V.fR1[q] = R1; V.fP1[q] = P1; V.fR2[q] = R2;
}

// regret key class: 2 no slot, 1 a single slot value, 0 otherwise (genetic.py:218-223)
__device__ __forceinline__ int r_class(const RepView &V, int q) {
  return V.fR1[q] < 0 ? 2 : (V.fC2[q] == CUDART_INF ? 1 : 0);
}
__device__ __forceinline__ double r_regret(const RepView &V, int q) {
  return r_class(V, q) == 0 ? V.fC2[q] - V.fC1[q] : 0.0;
}

__device__ __forceinline__ int r_len(const DevInst &I, int k) { return k + (I.open ? 1 : 2); }

// pref (left fold) and suf (right fold) of route r; lane 0 / lane 1 of a warp
__device__ void r_rebuild(const DevInst &I, const RepView &V, int r, int lane) {
  const int4 mt = V.rm[r];
  const int n = r_len(I, mt.x);
  const int *sq = V.seq + (size_t)r * V.Kp;
  RAt *pre = V.pre + (size_t)r * V.Kp, *suf = V.suf + (size_t)r * V.Kp;
  if (lane == 0) {
    RAt a = r_single(I, sq[0]);
    pre[0] = a;
    for (int i = 1; i < n; i++) {
      a = r_cat(I, a, sq[i - 1], r_single(I, sq[i]), sq[i]);
      pre[i] = a;
    }
  } else if (lane == 1) {
    RAt a = r_single(I, sq[n - 1]);
    suf[n - 1] = a;
    for (int i = n - 2; i >= 0; i--) {
      a = r_cat(I, r_single(I, sq[i]), sq[i], a, sq[i + 1]);
      suf[i] = a;
    }
  }
}

// route-local scan of every slot of route r for `node` (_best_slot restricted to r)
__device__ void r_scan(const DevInst &I, const RepView &V, int r, int node, bool feas_only, const double lam[4],
                       double &m1, int &pos1, double &m2) {
  const int4 mt = V.rm[r];
  const int k = mt.x, n = r_len(I, k);
  const int *sq = V.seq + (size_t)r * V.Kp;
  const RAt *pre = V.pre + (size_t)r * V.Kp, *suf = V.suf + (size_t)r * V.Kp;
  double o[4];
  r_terms(I, pre[n - 1], o);
  const RAt sn = r_single(I, node);
  m1 = CUDART_INF;
  m2 = CUDART_INF;
  pos1 = -1;
  for (int pos = 0; pos <= k; pos++) {
    RAt a = r_cat(I, pre[pos], sq[pos], sn, node);
    if (pos + 1 < n) a = r_cat(I, a, node, suf[pos + 1], sq[pos + 1]);
    double x[4];
    r_terms(I, a, x);
    const double dd = x[0] - o[0];
    double cost;
    if (feas_only) {
      if (!r_feasible(I, a)) continue;
      cost = dd;
    } else {
      cost = ((dd + lam[0] * (x[1] - o[1])) + lam[1] * (x[2] - o[2])) + lam[2] * (x[3] - o[3]);
    }
    if (cost < m1) {
      m2 = m1;
      m1 = cost;
      pos1 = pos;
    } else if (cost < m2) {
      m2 = cost;
    }
  }
}

__device__ __forceinline__ unsigned long long ord_d(double x) {  // order-preserving, -0 == +0
  unsigned long long u = (unsigned long long)__double_as_longlong(x + 0.0);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

constexpr int RP_THREADS = 256;
constexpr int RP_MAXND = 256;

__global__ void __launch_bounds__(RP_THREADS) k_repair(DevInst I, DevPop P, int B, int op, const int *pend_off,
                                                       const int *pend, RAt *g_pre, RAt *g_suf, double *g_c1,
                                                       double *g_c2, int *g_p1, double *g_fold, int *g_foldi,
                                                       int Pcap, int *status, long long *stats) {
  const int b = blockIdx.x;
  if (b >= B) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = RP_THREADS / 32;
  RepView V;
  V.Kp = P.Kp; V.J = P.J; V.K = P.K; V.Pcap = Pcap;
  V.seq = P.seq + (size_t)b * P.J * P.Kp;
  V.rm = P.rmeta + (size_t)b * P.J;
  V.pre = g_pre + (size_t)b * P.J * P.Kp;
  V.suf = g_suf + (size_t)b * P.J * P.Kp;
  V.c1 = g_c1 + (size_t)b * Pcap * P.J;
  V.c2 = g_c2 + (size_t)b * Pcap * P.J;
  V.p1 = g_p1 + (size_t)b * Pcap * P.J;
  V.fC1 = g_fold + (size_t)b * Pcap * 2;
  V.fC2 = V.fC1 + Pcap;
  V.fR1 = g_foldi + (size_t)b * Pcap * 3;
  V.fP1 = V.fR1 + Pcap;
  V.fR2 = V.fP1 + Pcap;
  const bool feas_only = op == 0 || op == 2, regret = op == 2 || op == 3;
  const int q0 = pend_off[b], P0 = pend_off[b + 1] - q0;
  const int *pd = pend + q0;
  const int *LOC = P.loc + (size_t)b * P.N;

  __shared__ int s_m, s_alive, s_err, s_needj, s_needk, s_touch, s_slots;
  __shared__ int s_cls, s_q;
  __shared__ unsigned long long s_key;
  __shared__ int s_cnt[RP_MAXND];
  __shared__ unsigned char s_dead[4096];
  __shared__ unsigned long long s_ev_dev;
  double lam[4];
  for (int i = 0; i < 4; i++) lam[i] = P.lam[b * 4 + i];

  if (tid == 0) {
    s_m = P.m[b];
    s_alive = P0;
    s_err = 0;
    s_needj = s_needk = 0;
    s_ev_dev = 0;
  }
  for (int q = tid; q < P0; q += RP_THREADS) {
    s_dead[q] = 0;
    const int v = pd[q];
    if (v < I.ND || v >= I.N || LOC[v] >= 0 || (q > 0 && pd[q - 1] >= v)) atomicExch(&s_err, MDR_ERR_ARG);
  }
  __syncthreads();
  if (s_err) {
    if (tid == 0) status[b] = s_err;
    return;
  }
  // open_route (genetic.py:148-166): depot of minimal (not free, cost, d)
  auto open_route = [&](int node) -> int {  // thread 0 only; returns the new route or -1
    const int m = s_m;
    if (m >= V.J) { s_needj = m + 1; return -1; }
    int best = -1, bnf = 0;
    double bcost = 0.0;
    for (int d = 0; d < I.ND; d++) {
      const double cost = I.dist[(size_t)d * I.N + node] + (I.open ? 0.0 : I.dist[(size_t)node * I.N + d]);
      const int nf = !(!I.nv_on || (double)s_cnt[d] < I.NV);
      if (best < 0 || nf < bnf || (nf == bnf && cost < bcost)) { best = d; bnf = nf; bcost = cost; }
    }
    int *sq = V.seq + (size_t)m * V.Kp;
    sq[0] = best;
    sq[1] = node;
    if (!I.open) sq[2] = best;
    V.rm[m] = make_int4(1, best, best, 0);
    s_cnt[best]++;
    s_m = m + 1;
    return m;
  };
  auto count_depots = [&]() {
    for (int d = tid; d < I.ND; d += RP_THREADS) s_cnt[d] = 0;
    __syncthreads();
    for (int r = tid; r < s_m; r += RP_THREADS) {
      const int4 mt = V.rm[r];
      if (mt.x > 0) atomicAdd(&s_cnt[mt.y], 1);
    }
    __syncthreads();
  };
  count_depots();
  if (!feas_only && s_m == 0 && P0 > 0) {  // degenerate guard of the relaxed modes (genetic.py:211-212)
    if (tid == 0) {
      if (open_route(pd[0]) < 0) s_err = MDR_ERR_CAPACITY;
      s_dead[0] = 1;
      s_alive = P0 - 1;
    }
    __syncthreads();
  }
  // prefix/suffix of every route: one warp per route (lane 0 prefix, lane 1 suffix)
  for (int r = wid; r < s_m; r += nw) r_rebuild(I, V, r, lane);
  __syncthreads();
  // all columns
  {
    const int m = s_m;
    for (long long it = tid; it < (long long)P0 * m; it += RP_THREADS) {
      const int q = (int)(it / m), r = (int)(it - (long long)q * m);
      if (s_dead[q]) continue;
      double m1, m2;
      int pos1;
      r_scan(I, V, r, pd[q], feas_only, lam, m1, pos1, m2);
      V.c1[(size_t)q * V.J + r] = m1;
      V.c2[(size_t)q * V.J + r] = m2;
      V.p1[(size_t)q * V.J + r] = pos1;
    }
  }
  __syncthreads();
  // per-customer fold of the route summaries (the state of _best_slot after the
  // whole scan): C1 at (R1, POS1), C2 from route R2 (-1: no second value)
  for (int q = tid; q < P0; q += RP_THREADS)
    if (!s_dead[q]) r_fold(V, q, s_m);
  if (tid == 0) {
    int slots = 0;
    for (int r = 0; r < s_m; r++) slots += V.rm[r].x + 1;
    s_slots = slots;
  }
  __syncthreads();
  long long ev_dev = 0, ev_ref = 0;
  while (s_alive > 0 && !s_err) {
    if (tid == 0) {
      s_cls = regret ? -1 : 0;
      s_key = regret ? 0ull : ~0ull;
      s_q = 0x7fffffff;
      ev_ref += (long long)s_alive * s_slots;
    }
    __syncthreads();
    // (a)/(b) the chosen customer: best = minimal C1, then smallest id; regret =
    // maximal (class, C2 - C1), then smallest id (keys (cls, val, -node), genetic.py:214-231)
    if (regret) {
      for (int q = tid; q < P0; q += RP_THREADS)
        if (!s_dead[q]) atomicMax(&s_cls, r_class(V, q));
      __syncthreads();
      for (int q = tid; q < P0; q += RP_THREADS)
        if (!s_dead[q] && r_class(V, q) == s_cls) atomicMax(&s_key, ord_d(r_regret(V, q)));
      __syncthreads();
      for (int q = tid; q < P0; q += RP_THREADS)
        if (!s_dead[q] && r_class(V, q) == s_cls && ord_d(r_regret(V, q)) == s_key) atomicMin(&s_q, q);
    } else {
      for (int q = tid; q < P0; q += RP_THREADS)
        if (!s_dead[q] && V.fR1[q] >= 0) atomicMin(&s_key, ord_d(V.fC1[q]));
      __syncthreads();
      for (int q = tid; q < P0; q += RP_THREADS)
        if (!s_dead[q] && V.fR1[q] >= 0 && ord_d(V.fC1[q]) == s_key) atomicMin(&s_q, q);
    }
    __syncthreads();
    if (tid == 0) {
      int q = s_q;
      int R = -1, POS = -1;
      if (q == 0x7fffffff) {  // best modes: no customer has a slot -> first pending, new route
        q = 0;
        while (s_dead[q]) q++;
      } else {
        R = V.fR1[q];
        POS = V.fP1[q];
      }
      s_dead[q] = 1;
      s_alive--;
      const int node = pd[q];
      if (R < 0) {
        const int r = open_route(node);
        if (r < 0) s_err = MDR_ERR_CAPACITY;
        s_touch = r;
        s_slots += 2;
      } else {
        int4 mt = V.rm[R];
        if (mt.x >= V.K) {
          s_needk = mt.x + 1;
          s_err = MDR_ERR_CAPACITY;
        } else {
          int *sq = V.seq + (size_t)R * V.Kp;
          const int n = r_len(I, mt.x);
          for (int i = n; i > POS + 1; i--) sq[i] = sq[i - 1];  // shifts the arrive depot too
          sq[POS + 1] = node;
          if (mt.x == 0) s_cnt[mt.y]++;
          mt.x += 1;
          V.rm[R] = mt;
        }
        s_touch = R;
        s_slots += 1;
      }
    }
    __syncthreads();
    if (s_err) break;
    const int rt = s_touch, m = s_m;
    if (wid == 0) r_rebuild(I, V, rt, lane);
    __syncthreads();
    // (e) the touched route's column for every pending customer; refold a
    // customer only when its top two can change: rt supplied C1 or C2, or the
    // new minimum of rt reaches C2 (otherwise every value of rt is > C2 before
    // and after, and the first minimum lies in another route)
    const int kk = V.rm[rt].x + 1;
    for (int q = tid; q < P0; q += RP_THREADS) {
      if (s_dead[q]) continue;
      double m1, m2;
      int pos1;
      r_scan(I, V, rt, pd[q], feas_only, lam, m1, pos1, m2);
      V.c1[(size_t)q * V.J + rt] = m1;
      V.c2[(size_t)q * V.J + rt] = m2;
      V.p1[(size_t)q * V.J + rt] = pos1;
      ev_dev += kk;
      if (V.fR1[q] == rt || V.fR2[q] == rt || !(m1 > V.fC2[q])) r_fold(V, q, m);
    }
    __syncthreads();
  }
  atomicAdd(&s_ev_dev, (unsigned long long)ev_dev);
  __syncthreads();
  if (tid == 0) {
    P.m[b] = s_m;
    status[b] = s_err;
    stats[3 * b + 0] = (long long)s_ev_dev;
    stats[3 * b + 1] = ev_ref;
    stats[3 * b + 2] = ((long long)s_needj << 32) | (unsigned)s_needk;
  }
}

void launch_repair(const DevInst &I, const DevPop &P, int B, int op, const int *pend_off, const int *pend,
                   void *pre, void *suf, double *c1, double *c2, int *p1, double *fold, int *foldi, int Pcap,
                   int *status, long long *stats, cudaStream_t s) {
  if (B <= 0) return;
  k_repair<<<B, RP_THREADS, 0, s>>>(I, P, B, op, pend_off, pend, (RAt *)pre, (RAt *)suf, c1, c2, p1, fold, foldi,
                                    Pcap, status, stats);
}

size_t repair_attr_bytes() { return sizeof(RAt); }

// ---------------------------------------------------------------------------
// Initial solutions (genetic.initial_solution, genetic.py:251-294), one CTA per
// individual.  Depot by depot (id order), the depot's members are inserted in
// the given (caller-shuffled) order: every route of the depot is scanned by a
// warp with r_scan in feasible-only mode (cost = route distance increase of
// the _attr_feasible candidates, genetic.py:109-116, 271-279), the first minimum
// over (route, position) in scan order wins (strict '<', as the reference's
// nested loop), else a new route (d, d, [c]) while the depot's fleet allows,
// else the customer is left over.  The depot's routes are appended to the
// individual's route list (sol.routes.extend order); pre/suf hold only the
// current depot's routes (indexed from its first route).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(RP_THREADS) k_construct(DevInst I, DevPop P, int B, const int *ooff,
                                                          const int *order, RAt *g_pre, RAt *g_suf, int Jd,
                                                          int *n_left, int *left, int *status) {
  const int b = blockIdx.x;
  if (b >= B) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = RP_THREADS / 32;
  __shared__ double s_m1[RP_THREADS / 32];
  __shared__ int s_r[RP_THREADS / 32], s_p[RP_THREADS / 32];
  __shared__ int s_m, s_r0, s_nl, s_err, s_touch;
  if (tid == 0) { s_m = 0; s_nl = 0; s_err = 0; }
  __syncthreads();
  const double lam0[4] = {0.0, 0.0, 0.0, 0.0};
  for (int d = 0; d < I.ND && !s_err; d++) {
    if (tid == 0) s_r0 = s_m;
    __syncthreads();
    RepView V;
    V.Kp = P.Kp; V.J = P.J; V.K = P.K;
    V.seq = P.seq + ((size_t)b * P.J + s_r0) * P.Kp;  // this depot's routes, local index 0..
    V.rm = P.rmeta + (size_t)b * P.J + s_r0;
    V.pre = g_pre + (size_t)b * Jd * P.Kp;
    V.suf = g_suf + (size_t)b * Jd * P.Kp;
    const int o0 = ooff[b * I.ND + d], o1 = ooff[b * I.ND + d + 1];
    for (int t = o0; t < o1; t++) {
      const int cst = order[t];
      const int md = s_m - s_r0;
      // per thread: first minimum over its routes (increasing route order), then
      // the warp's minimum by (cost, route)
      double bm = CUDART_INF;
      int br = -1, bp = -1;
      for (int r = tid; r < md; r += RP_THREADS) {
        double m1, m2;
        int p1;
        r_scan(I, V, r, cst, true, lam0, m1, p1, m2);
        if (p1 >= 0 && m1 < bm) { bm = m1; br = r; bp = p1; }
      }
#pragma unroll
      for (int sh = 16; sh > 0; sh >>= 1) {
        const double om = __shfl_xor_sync(0xffffffffu, bm, sh);
        const int orr = __shfl_xor_sync(0xffffffffu, br, sh), op = __shfl_xor_sync(0xffffffffu, bp, sh);
        if (orr >= 0 && (br < 0 || om < bm || (om == bm && orr < br))) { bm = om; br = orr; bp = op; }
      }
      if (lane == 0) { s_m1[wid] = bm; s_r[wid] = br; s_p[wid] = bp; }
      __syncthreads();
      if (tid == 0) {
        // fold the warps' minima by (cost, route): the reference's scan order
        double cm = CUDART_INF;
        int cr = -1, cp = -1;
        for (int w = 0; w < nw; w++) {
          if (s_r[w] < 0) continue;
          if (s_m1[w] < cm || (s_m1[w] == cm && s_r[w] < cr)) { cm = s_m1[w]; cr = s_r[w]; cp = s_p[w]; }
        }
        s_touch = -1;
        if (cr >= 0) {
          int4 mt = V.rm[cr];
          if (mt.x >= V.K) {
            s_err = MDR_ERR_CAPACITY;
          } else {
            int *sq = V.seq + (size_t)cr * V.Kp;
            const int n = r_len(I, mt.x);
            for (int i = n; i > cp + 1; i--) sq[i] = sq[i - 1];
            sq[cp + 1] = cst;
            mt.x += 1;
            V.rm[cr] = mt;
            s_touch = cr;
          }
        } else if (!I.nv_on || (double)md < I.NV) {
          if (s_m >= P.J || md >= Jd) {
            s_err = MDR_ERR_CAPACITY;
          } else {
            int *sq = V.seq + (size_t)md * V.Kp;
            sq[0] = d;
            sq[1] = cst;
            if (!I.open) sq[2] = d;
            V.rm[md] = make_int4(1, d, d, 0);
            s_m += 1;
            s_touch = md;
          }
        } else {
          left[(size_t)b * (I.N - I.ND) + s_nl++] = cst;
        }
      }
      __syncthreads();
      if (s_err) break;
      if (s_touch >= 0 && wid == 0) r_rebuild(I, V, s_touch, lane);
      __syncthreads();
    }
    __syncthreads();
  }
  if (tid == 0) {
    P.m[b] = s_m;
    n_left[b] = s_nl;
    status[b] = s_err;
  }
}

void launch_construct(const DevInst &I, const DevPop &P, int B, const int *ooff, const int *order, void *pre,
                      void *suf, int Jd, int *n_left, int *left, int *status, cudaStream_t s) {
  if (B <= 0) return;
  k_construct<<<B, RP_THREADS, 0, s>>>(I, P, B, ooff, order, (RAt *)pre, (RAt *)suf, Jd, n_left, left, status);
}

// evaluation.evaluate (evaluation.py:206-224) of every uploaded individual, with
// the scalar algebra's semantics: each route folded left with Python max/min
// (route_attr), route_contributions per route, then D/V1/V2/V3 summed in route
// order skipping empty routes, V4 = theta * (closures + fleet excess) and
// F = D + l0 V1 + l1 V2 + l2 V3 + l3 V4.  out[b] = {D, V1, V2, V3, V4, F}.
__global__ void __launch_bounds__(128) k_breakdown(DevInst I, DevPop P, int B, const double *lam, double *rt,
                                                   double *out) {
  const int b = blockIdx.x;
  if (b >= B) return;
  const int m = P.m[b];
  const int4 *RM = P.rmeta + (size_t)b * P.J;
  double *T = rt + (size_t)b * P.J * 5;
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    const int4 mt = RM[r];
    if (mt.x == 0) continue;
    const int *sq = P.seq + ((size_t)b * P.J + r) * P.Kp;
    const int n = mt.x + (I.open ? 1 : 2);
    RAt a = r_single(I, sq[0]);
    for (int i = 1; i < n; i++) a = r_cat(I, a, sq[i - 1], r_single(I, sq[i]), sq[i]);
    double o[4];
    r_terms(I, a, o);
    T[r * 5 + 0] = o[0];
    T[r * 5 + 1] = o[1];
    T[r * 5 + 2] = o[2];
    T[r * 5 + 3] = o[3];
    T[r * 5 + 4] = I.open ? 0.0 : (mt.y != mt.z ? 1.0 : 0.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double D = 0.0, V1 = 0.0, V2 = 0.0, V3 = 0.0, clo = 0.0;
    int cnt[RP_MAXND];
    for (int d = 0; d < I.ND; d++) cnt[d] = 0;
    for (int r = 0; r < m; r++) {
      const int4 mt = RM[r];
      if (mt.x == 0) continue;
      D += T[r * 5 + 0];
      V1 += T[r * 5 + 1];
      V2 += T[r * 5 + 2];
      V3 += T[r * 5 + 3];
      clo += T[r * 5 + 4];
      cnt[mt.y]++;
    }
    double ex = 0.0;
    if (I.nv_on)
      for (int d = 0; d < I.ND; d++) ex += py_max((double)cnt[d] - I.NV, 0.0);
    const double V4 = I.theta * (clo + ex);
    const double *l = lam + 4 * (size_t)b;
    double *o = out + 6 * (size_t)b;
    o[0] = D; o[1] = V1; o[2] = V2; o[3] = V3; o[4] = V4;
    o[5] = (((D + l[0] * V1) + l[1] * V2) + l[2] * V3) + l[3] * V4;
  }
}

// route_attr (evaluation.py:97-106) of every route of individuals b0 .. b0+nb-1: the
// scalar left fold with Python max/min; out[(b - b0) * J + r] = {dist, load, T, E, L, TW}
__global__ void k_route_attrs(DevInst I, DevPop P, int b0, int nb, double *out) {
  const int b = b0 + blockIdx.x;
  if (blockIdx.x >= nb) return;
  const int m = P.m[b];
  const int4 *RM = P.rmeta + (size_t)b * P.J;
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    const int4 mt = RM[r];
    const int *sq = P.seq + ((size_t)b * P.J + r) * P.Kp;
    const int n = mt.x + (I.open ? 1 : 2);
    RAt a = r_single(I, sq[0]);
    for (int i = 1; i < n; i++) a = r_cat(I, a, sq[i - 1], r_single(I, sq[i]), sq[i]);
    double *o = out + ((size_t)blockIdx.x * P.J + r) * 6;
    o[0] = a.dist; o[1] = a.load; o[2] = a.T; o[3] = a.E; o[4] = a.L; o[5] = a.TW;
  }
}

void launch_route_attrs(const DevInst &I, const DevPop &P, int b0, int nb, double *out, cudaStream_t s) {
  if (nb > 0) k_route_attrs<<<nb, 128, 0, s>>>(I, P, b0, nb, out);
}

void launch_breakdown(const DevInst &I, const DevPop &P, int B, const double *lam, double *rt, double *out,
                      cudaStream_t s) {
  if (B <= 0) return;
  k_breakdown<<<B, 128, 0, s>>>(I, P, B, lam, rt, out);
}

}  // namespace mdr
