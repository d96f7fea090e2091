// mdr_device.cuh -- device-side data layout and fp64 primitives of the
// sm_100a local search.  Compiled with -fmad=false: no FMA contraction, so
// every expression keeps the rounding of the reference's numpy expression.
//
// HBM layout (per GPU, library-owned):
//   instance : dist/time [N*N] f64, node {q,s,e,l} [N] double4,
//              lists [NC*W] i32 (customer rows only)
//   population, individual b (strides J routes, Kp = K+2 sequence slots):
//     m[b]                       route count
//     rmeta[b][r]  int4          {k, depart, arrive, closure flag}
//     seq[b][r][Kp] i32          sequence positions (depot, customers, [arrive])
//     loc[b][node] i32           (route << 9) | customer index, -1 unrouted
//     rcon[b][r]   double4       route D (raw table value), V1, V2, V3
//     tabP/tabS[b][r][Kp][FE]    prefix (0..j) / suffix (i..n-1) subsequence
//                                attributes = left folds, batch.py:85-124
//     fleet[b][d]  double2       fleet_inc, fleet_dec (batch.py:149-158)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define MDR_CHUNK 256

// k_eval_c shapes (DevPop::ct selects one per population): small populations /
// instances -- 8 warps, 8 items per CTA task, 2 CTAs per SM (more, smaller tasks
// for an under-filled GPU); large -- 16 warps, 32 items per task (2 per warp),
// 1 CTA per SM (the route staging amortised over twice the items).  Measured:
// C2 7.9 vs 7.3 G/s, C3 8.4 vs 6.6 (small wins); C4 22.8 vs 22.3, C5 25.2 vs 23.8
// (large wins).
#ifndef MDR_SMALL_CU
#define MDR_SMALL_CU 8
#endif
#ifndef MDR_SMALL_CT
#define MDR_SMALL_CT 8
#endif
#ifndef MDR_LARGE_CU
#define MDR_LARGE_CU 16
#endif
#ifndef MDR_EVAL_OCC
#define MDR_EVAL_OCC 16  // warps per SM the staged evaluators are register-budgeted for (launch bounds)
#endif
#ifndef MDR_LARGE_CT
#define MDR_LARGE_CT 32
#endif

#define MDR_EPS 1e-9

namespace mdr {

struct DevInst {
  int N, ND, NC, W;
  const double *dist, *time;
  int talias;
  const double4 *node;  // {demand, service, tw_early, tw_late}
  const int *lists;     // [NC][W]
  double Q, Dmax, NV;
  int d_on, nv_on, open, win;
  double gamma, theta;
  double rQ, rD;  // RN(1/Q), RN(1/Dmax) for div_q (host IEEE division)
  int sym;        // dist (and time) exactly symmetric: m[x][y] == m[y][x] bit for bit
};

// per-individual search state (localsearch.py:107-140 loop variables)
struct LsState {
  int pass, pos, any, accepted;
  int done, status, op_evals, n_feasible;
  int n_improving, pad0;
  long long moves_applied;
  double bestD;
  int need_f, need_g, need_j, need_k;  // capacity a retry needs (status 3)
};

struct DevPop {
  int Bcap, J, K, Kp, Fcap, FE;
  int staged;  // relocate/swap/2-opt* use the CTA-staged evaluators (mdr_staged.cuh)
  int ct;      // items per CTA task of the staged evaluators (MDR_SMALL_CT / MDR_LARGE_CT)
  int tsplit;  // sub-tasks per customer block (relocate boundary family, flattened swap): 1, 2 or 4
  int N, ND;
  int *m;
  int4 *rmeta;
  int *seq;
  int *loc;
  int *nxs;  // [B][N] node after this customer in its route's sequence (arrive depot), -1 past the end
  double4 *rcon;
  double *tabP, *tabS;
  double *tabT;  // [B][J][Kp][Kp][FE] full subsequence table (i..j), left fold from i
  double2 *fleet;
  double *fexcess;
  double *lam;
  // local-search bookkeeping
  LsState *st;
  unsigned long long *cands;  // [B][6]
  const uint8_t *perms;       // [B][maxp][nops]
  int maxp, nops;
  // round scratch
  int *op_cur;                // [B]
  int *wsize;                 // [B]
  int *chunk_off;             // [B+1]
  int *total_chunks;          // [1]
  int *active;                // [1]
  int *task_next;             // [8] dynamic task counters: per operator, [6] relocate boundary family (split)
  int *opcnt;                 // [6] individuals evaluating each operator this round
  int *optasks;               // [6] tasks per operator this round
  int *opb;                   // [6][Bcap] individual ids per operator
  int *opoff;                 // [6][Bcap+1] first task of each individual within its operator
  ulonglong2 *leader;         // [B] running min {ord(dF), key} of the round
  ulonglong2 *gq;             // [Gcap] generic-path queue {key, b | op << 24}; region r = [gbase[r], gbase[r+1]):
                              // overlap mode: 0 = 2-opt/depot ops, 1 = intra-route relocate, 2 = intra-route
                              // swap, each drained right behind its producer; otherwise region 1 holds all
  int *gcount;                // [3] entries queued per region
  int Gcap;
  int gbase[4];
  int *tcount;                // [max tasks] candidates per task
  ulonglong2 *partial;        // [max tasks] {ord(dF), key}
  ulonglong2 *fol;            // [B][Fcap]
  int *fcount;                // [B]
  int *nanflag;               // [B]
  int *scratch_seq;           // [B][J][Kp]
  int4 *scratch_meta;         // [B][J]
  // accepted-step trace (on_feasible replay): per individual [tcap] words, trcount used
  unsigned long long *trace;
  long long *trcount;
  long long tcap;
  // best-feasible snapshot
  int *best_m;
  int4 *best_meta;
  int *best_seq;
};

struct LsParams {
  int depth, multi_move;
  double kappa, lam_min, lam_max;
  int B;
  int snapshot;  // keep the best-feasible snapshot (for on_feasible)
  int trace;     // record every accepted step: {op<<56 | feasible<<55 | n moves, D bits, keys...}
};

// ---------------------------------------------------------------------------
// subsequence attributes (evaluation.SeqAttr, evaluation.py:22-57)
// ---------------------------------------------------------------------------
template <bool WIN>
struct At {
  double dist, load, T, E, L, TW;
  int first, last;
};

__device__ __forceinline__ double npmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double npmin(double a, double b) { return a < b ? a : b; }

template <bool WIN>
__device__ __forceinline__ At<WIN> a_empty() {
  At<WIN> a;
  a.dist = 0.0; a.load = 0.0; a.T = 0.0; a.E = 0.0; a.L = __longlong_as_double(0x7ff0000000000000ll); a.TW = 0.0;
  a.first = -1; a.last = -1;
  return a;
}

template <bool WIN>
__device__ __forceinline__ At<WIN> a_node(const DevInst &I, int v) {
  const double2 *np2 = reinterpret_cast<const double2 *>(I.node + v);
  double2 qs = __ldg(np2);
  At<WIN> a;
  a.dist = 0.0; a.load = qs.x; a.T = qs.y;
  if (WIN) {
    double2 el = __ldg(np2 + 1);
    a.E = el.x; a.L = el.y;
  } else {
    a.E = 0.0; a.L = 0.0;
  }
  a.TW = 0.0;
  a.first = v; a.last = v;
  return a;
}

// distance/time link a.last -> b.first.  When the matrices are exactly
// symmetric the caller may name the warp-uniform end so the read comes from
// that node's (L1-resident) row; the value is identical by symmetry.
struct Link {
  double c, t;
};
__device__ __forceinline__ Link link_of(const DevInst &I, int x, int y) {
  size_t lk = (size_t)x * (size_t)I.N + (size_t)y;
  Link L;
  L.c = __ldg(I.dist + lk);
  L.t = I.talias ? L.c : __ldg(I.time + lk);
  return L;
}
// link x -> y where y is warp-uniform
__device__ __forceinline__ Link link_to_u(const DevInst &I, int x, int y) {
  return I.sym ? link_of(I, y, x) : link_of(I, x, y);
}

// vconcat (batch.py:223-262) of two non-empty subsequences with a given link
template <bool WIN>
__device__ __forceinline__ At<WIN> a_cat_l(const At<WIN> &a, const At<WIN> &b, Link L) {
  const double c = L.c, t = L.t;
  At<WIN> o;
  o.dist = (a.dist + c) + b.dist;
  o.load = a.load + b.load;
  if (WIN) {
    double delta = (a.T - a.TW) + t;
    double wait = npmax((b.E - delta) - a.L, 0.0);
    double warp = npmax((a.E + delta) - b.L, 0.0);
    o.T = ((a.T + b.T) + t) + wait;
    o.TW = (a.TW + b.TW) + warp;
    o.E = npmax(b.E - delta, a.E) - wait;
    o.L = npmin(b.L - delta, a.L) + warp;
  } else {
    o.T = (a.T + b.T) + t;
    o.E = 0.0; o.L = 0.0; o.TW = 0.0;
  }
  o.first = a.first;
  o.last = b.last;
  return o;
}

template <bool WIN>
__device__ __forceinline__ At<WIN> a_cat_ne(const DevInst &I, const At<WIN> &a, const At<WIN> &b) {
  return a_cat_l<WIN>(a, b, link_of(I, a.last, b.first));
}

// vconcat with possibly empty operands: an empty side is the exact identity
template <bool WIN>
__device__ __forceinline__ At<WIN> a_cat(const DevInst &I, const At<WIN> &a, const At<WIN> &b) {
  if (b.first < 0) return a;
  if (a.first < 0) return b;
  return a_cat_ne<WIN>(I, a, b);
}

// Correctly rounded a / b for a divisor known in advance (rb = RN(1/b)):
// Markstein's correction q' = RN(q + r*rb), r = a - q*b exact (FMA), then an
// exact acceptance test: the remainder of q' is recomputed exactly and q' is
// accepted only if |a/b - q'| is strictly below half the smaller neighbour
// gap of q'; anything else (ties, specials, extreme exponents) falls back to
// the IEEE division.  The result is therefore always RN(a / b).
__device__ __forceinline__ double div_q(double a, double b, double rb) {
  double q = __dmul_rn(a, rb);
  double r = __fma_rn(-q, b, a);
  q = __fma_rn(r, rb, q);
  long long bits = __double_as_longlong(q);
  int e = (int)((bits >> 52) & 0x7ff);
  if (e > 60 && e < 2000) {
    double r2 = fabs(__fma_rn(-q, b, a));  // exact remainder of q
    // smaller neighbour gap: ulp(q), or ulp(q)/2 when |q| is a power of two
    long long ge = (bits & 0x000fffffffffffffll) ? (long long)(e - 52) : (long long)(e - 53);
    double gap = __longlong_as_double(ge << 52);
    if (__dmul_rn(2.0, r2) < __dmul_rn(gap, fabs(b))) return q;
  }
  return a / b;
}

// ---------------------------------------------------------------------------
// table access
// ---------------------------------------------------------------------------
__device__ __forceinline__ size_t row_base(const DevPop &P, int b, int r) {
  return ((size_t)b * P.J + r) * P.Kp;
}

template <bool WIN>
__device__ __forceinline__ At<WIN> tab_load(const DevPop &P, const double *tab, int b, int r, int i) {
  const double2 *e = reinterpret_cast<const double2 *>(tab + (row_base(P, b, r) + i) * P.FE);
  At<WIN> a;
  double2 x = e[0], y = e[1];
  a.dist = x.x; a.load = x.y; a.T = y.x;
  if (WIN) {
    double2 z = e[2];
    a.E = y.y; a.L = z.x; a.TW = z.y;
  } else {
    a.E = 0.0; a.L = 0.0; a.TW = 0.0;
  }
  return a;
}

template <bool WIN>
__device__ __forceinline__ void tab_store(const DevPop &P, double *tab, int b, int r, int i, const At<WIN> &a) {
  double2 *e = reinterpret_cast<double2 *>(tab + (row_base(P, b, r) + i) * P.FE);
  e[0] = make_double2(a.dist, a.load);
  if (WIN) {
    e[1] = make_double2(a.T, a.E);
    e[2] = make_double2(a.L, a.TW);
  } else {
    e[1] = make_double2(a.T, 0.0);
  }
}

template <bool WIN>
__device__ __forceinline__ void tab_store_at(double *p, const At<WIN> &a) {
  double2 *e = reinterpret_cast<double2 *>(p);
  e[0] = make_double2(a.dist, a.load);
  if (WIN) {
    e[1] = make_double2(a.T, a.E);
    e[2] = make_double2(a.L, a.TW);
  } else {
    e[1] = make_double2(a.T, 0.0);
  }
}

// attributes of sequence positions i..j of route r (SolutionCache.gather,
// batch.py:184-221); j < i is the empty sequence.  The source is the prefix
// table (i == 0), the suffix table (j == n-1) or the full table T[r][i][j] --
// all three hold the same left fold from i, bit for bit.
template <bool WIN>
__device__ __forceinline__ At<WIN> gat(const DevInst &I, const DevPop &P, int b, int r, int i, int j, int n) {
  if (j < i) return a_empty<WIN>();
  const size_t rb = row_base(P, b, r);
  const int *sq = P.seq + rb;
  // one load sequence from a selected source (no divergent per-table branches)
  const double *src = i == 0 ? P.tabP + (rb + j) * P.FE
                             : (j == n - 1 ? P.tabS + (rb + i) * P.FE : P.tabT + ((rb + i) * P.Kp + j) * P.FE);
  const double2 *e = reinterpret_cast<const double2 *>(src);
  At<WIN> a;
  double2 x = __ldg(e), y = __ldg(e + 1);
  a.dist = x.x; a.load = x.y; a.T = y.x;
  if (WIN) {
    double2 z = __ldg(e + 2);
    a.E = y.y; a.L = z.x; a.TW = z.y;
  } else {
    a.E = 0.0; a.L = 0.0; a.TW = 0.0;
  }
  a.first = __ldg(sq + i); a.last = __ldg(sq + j);
  return a;
}

template <bool WIN>
__device__ __forceinline__ void swap_ends(At<WIN> &a) {
  int t = a.first; a.first = a.last; a.last = t;
}

// _route_penalties (batch.py:271-293); zeros for an empty route
template <bool WIN>
__device__ __forceinline__ void contrib(const DevInst &I, const At<WIN> &a, int dep, int arr, int kc, double o[5]) {
  if (kc <= 0) { o[0] = o[1] = o[2] = o[3] = o[4] = 0.0; return; }
  o[0] = a.dist;
  o[1] = WIN ? I.gamma * a.TW : 0.0;
  double x = I.theta * npmax(a.load - I.Q, 0.0);
  o[2] = x == 0.0 ? 0.0 : div_q(x, I.Q, I.rQ);
  if (I.d_on) {
    double y = I.theta * npmax(a.T - I.Dmax, 0.0);
    o[3] = y == 0.0 ? 0.0 : div_q(y, I.Dmax, I.rD);
  } else {
    o[3] = 0.0;
  }
  o[4] = I.open ? 0.0 : (dep != arr ? 1.0 : 0.0);
}

// ---------------------------------------------------------------------------
// candidates, keys
// ---------------------------------------------------------------------------
struct Cand {
  int r1, p1, r2, p2, l1, l2, rev1, rev2, depot, mode;
};

// Move.key() order (moves.py:66-70) packed into 58 bits, -1 fields biased by 1
__host__ __device__ __forceinline__ unsigned long long pack_key(const Cand &c) {
  return ((unsigned long long)(c.r1 + 1) << 46) | ((unsigned long long)(c.r2 + 1) << 34) |
         ((unsigned long long)(c.p1 + 1) << 25) | ((unsigned long long)(c.p2 + 1) << 16) |
         ((unsigned long long)c.l1 << 14) | ((unsigned long long)c.l2 << 12) |
         ((unsigned long long)c.rev1 << 11) | ((unsigned long long)c.rev2 << 10) |
         ((unsigned long long)(c.depot + 1) << 2) | (unsigned long long)(c.mode + 1);
}

__host__ __device__ __forceinline__ Cand unpack_key(unsigned long long k) {
  Cand c;
  c.r1 = (int)((k >> 46) & 0xfff) - 1;
  c.r2 = (int)((k >> 34) & 0xfff) - 1;
  c.p1 = (int)((k >> 25) & 0x1ff) - 1;
  c.p2 = (int)((k >> 16) & 0x1ff) - 1;
  c.l1 = (int)((k >> 14) & 3);
  c.l2 = (int)((k >> 12) & 3);
  c.rev1 = (int)((k >> 11) & 1);
  c.rev2 = (int)((k >> 10) & 1);
  c.depot = (int)((k >> 2) & 0xff) - 1;
  c.mode = (int)(k & 3) - 1;
  return c;
}

// monotone map of a double onto uint64 (-0 canonicalised to +0)
__device__ __forceinline__ unsigned long long ord_of(double x) {
  x = x + 0.0;
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord(unsigned long long o) {
  unsigned long long u = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  return __longlong_as_double((long long)u);
}

struct Delta {
  double dD, dV1, dV2, dV3, dV4, dF;
  int fn;
};

// evaluate_candidates (batch.py:365-553) for one candidate of individual b.
// FOP >= 0 fixes the operator and SAME the same-route case at compile time
// (the intra-route queue regions), so only that branch is generated.
template <bool WIN, int FOP = -1, bool SAME = false>
__device__ __forceinline__ Delta eval_cand(const DevInst &I, const DevPop &P, int b, int op, const Cand &c,
                                           const double lam[4]) {
  if (FOP >= 0) op = FOP;
  double nw[5], cA[5], cB[5];
  double fleet_delta = 0.0;
  int fn = 1, two = 0;
  const int4 *RM = P.rmeta + (size_t)b * P.J;
  const double2 *FL = P.fleet + (size_t)b * P.ND;
  int4 m1 = RM[c.r1];
  int k1 = m1.x, n1 = k1 + (I.open ? 1 : 2);
  int r1 = c.r1, r2 = c.r2, p1 = c.p1, p2 = c.p2, l1 = c.l1, l2 = c.l2;
  switch (op) {
    case 0: {  // RELOCATE batch.py:391-428
      At<WIN> seg = gat<WIN>(I, P, b, r1, p1 + 1, p1 + l1, n1);
      if (c.rev1) swap_ends(seg);
      if (SAME || r1 == r2) {
        bool before = p2 <= p1;
        At<WIN> x = gat<WIN>(I, P, b, r1, 0, before ? p2 : p1, n1);
        At<WIN> mid = before ? gat<WIN>(I, P, b, r1, p2 + 1, p1, n1) : gat<WIN>(I, P, b, r1, p1 + l1 + 1, p2, n1);
        if (before) { x = a_cat<WIN>(I, x, seg); x = a_cat<WIN>(I, x, mid); }
        else { x = a_cat<WIN>(I, x, mid); x = a_cat<WIN>(I, x, seg); }
        x = a_cat<WIN>(I, x, gat<WIN>(I, P, b, r1, before ? p1 + l1 + 1 : p2 + 1, n1 - 1, n1));
        contrib<WIN>(I, x, m1.y, m1.z, k1, cA);
        for (int f = 0; f < 5; f++) nw[f] = 0.0 + cA[f];
      } else {
        two = 1;
        int4 m2 = RM[r2];
        int k2 = m2.x, n2 = k2 + (I.open ? 1 : 2);
        At<WIN> A = a_cat<WIN>(I, gat<WIN>(I, P, b, r1, 0, p1, n1), gat<WIN>(I, P, b, r1, p1 + l1 + 1, n1 - 1, n1));
        At<WIN> B = a_cat<WIN>(I, gat<WIN>(I, P, b, r2, 0, p2, n2), seg);
        B = a_cat<WIN>(I, B, gat<WIN>(I, P, b, r2, p2 + 1, n2 - 1, n2));
        int kA = k1 - l1, kB = k2 + l1;
        contrib<WIN>(I, A, m1.y, m1.z, kA, cA);
        contrib<WIN>(I, B, m2.y, m2.z, kB, cB);
        for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
        if (I.nv_on && kA == 0) { fleet_delta = 0.0 + FL[m1.y].y; fn = 0; }
      }
      break;
    }
    case 1: {  // SWAP batch.py:430-463
      At<WIN> segA = gat<WIN>(I, P, b, r1, p1 + 1, p1 + l1, n1);
      if (c.rev1) swap_ends(segA);
      if (SAME || r1 == r2) {
        At<WIN> segB = gat<WIN>(I, P, b, r1, p2 + 1, p2 + l2, n1);
        if (c.rev2) swap_ends(segB);
        At<WIN> x = a_cat<WIN>(I, gat<WIN>(I, P, b, r1, 0, p1, n1), segB);
        x = a_cat<WIN>(I, x, gat<WIN>(I, P, b, r1, p1 + l1 + 1, p2, n1));
        x = a_cat<WIN>(I, x, segA);
        x = a_cat<WIN>(I, x, gat<WIN>(I, P, b, r1, p2 + l2 + 1, n1 - 1, n1));
        contrib<WIN>(I, x, m1.y, m1.z, k1, cA);
        for (int f = 0; f < 5; f++) nw[f] = 0.0 + cA[f];
      } else {
        two = 1;
        int4 m2 = RM[r2];
        int k2 = m2.x, n2 = k2 + (I.open ? 1 : 2);
        At<WIN> segB = gat<WIN>(I, P, b, r2, p2 + 1, p2 + l2, n2);
        if (c.rev2) swap_ends(segB);
        At<WIN> A = a_cat<WIN>(I, gat<WIN>(I, P, b, r1, 0, p1, n1), segB);
        A = a_cat<WIN>(I, A, gat<WIN>(I, P, b, r1, p1 + l1 + 1, n1 - 1, n1));
        At<WIN> B = a_cat<WIN>(I, gat<WIN>(I, P, b, r2, 0, p2, n2), segA);
        B = a_cat<WIN>(I, B, gat<WIN>(I, P, b, r2, p2 + l2 + 1, n2 - 1, n2));
        contrib<WIN>(I, A, m1.y, m1.z, k1 - l1 + l2, cA);
        contrib<WIN>(I, B, m2.y, m2.z, k2 - l2 + l1, cB);
        for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
      }
      break;
    }
    case 3: {  // TWO_OPT batch.py:465-473
      At<WIN> seg = gat<WIN>(I, P, b, r1, p1 + 1, p2 + 1, n1);
      swap_ends(seg);
      At<WIN> x = a_cat<WIN>(I, gat<WIN>(I, P, b, r1, 0, p1, n1), seg);
      x = a_cat<WIN>(I, x, gat<WIN>(I, P, b, r1, p2 + 2, n1 - 1, n1));
      contrib<WIN>(I, x, m1.y, m1.z, k1, cA);
      for (int f = 0; f < 5; f++) nw[f] = 0.0 + cA[f];
      break;
    }
    case 2: {  // TWO_OPT_STAR batch.py:475-494
      two = 1;
      int4 m2 = RM[r2];
      int k2 = m2.x, n2 = k2 + (I.open ? 1 : 2);
      At<WIN> A = a_cat<WIN>(I, gat<WIN>(I, P, b, r1, 0, p1, n1), gat<WIN>(I, P, b, r2, p2 + 1, n2 - 1, n2));
      At<WIN> B = a_cat<WIN>(I, gat<WIN>(I, P, b, r2, 0, p2, n2), gat<WIN>(I, P, b, r1, p1 + 1, n1 - 1, n1));
      int kA = p1 + (k2 - p2), kB = p2 + (k1 - p1);
      contrib<WIN>(I, A, m1.y, m2.z, kA, cA);
      contrib<WIN>(I, B, m2.y, m1.z, kB, cB);
      for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
      if (I.nv_on) {
        fleet_delta = (0.0 + (kA == 0 ? FL[m1.y].y : 0.0)) + (kB == 0 ? FL[m2.y].y : 0.0);
        fn = (kA > 0) && (kB > 0);
      }
      break;
    }
    case 4: {  // DEPOT_INSERT batch.py:496-517
      int d = c.depot;
      At<WIN> head = gat<WIN>(I, P, b, r1, 0, p1, n1), tail;
      if (!I.open) {
        head = a_cat<WIN>(I, head, a_node<WIN>(I, m1.z));
        tail = a_cat<WIN>(I, a_node<WIN>(I, d), gat<WIN>(I, P, b, r1, p1 + 1, k1, n1));
        tail = a_cat<WIN>(I, tail, a_node<WIN>(I, d));
      } else {
        tail = a_cat<WIN>(I, a_node<WIN>(I, d), gat<WIN>(I, P, b, r1, p1 + 1, k1, n1));
      }
      contrib<WIN>(I, head, m1.y, m1.z, p1, cA);
      contrib<WIN>(I, tail, d, d, k1 - p1, cB);
      for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
      if (I.nv_on) {
        bool drops = p1 == 0, same_dep = d == m1.y;
        double fd = (drops && same_dep) ? 0.0 : (drops ? FL[d].x + FL[m1.y].y : FL[d].x);
        fleet_delta = 0.0 + fd;
        fn = 0;
      }
      break;
    }
    default: {  // DEPOT_REPLACE batch.py:519-540
      int d = c.depot, mode = c.mode;
      int dep_new = mode != 1 ? d : m1.y;
      int arr_new = mode != 0 ? d : m1.z;
      At<WIN> x0 = mode == 1 ? a_empty<WIN>() : a_node<WIN>(I, dep_new);
      int i0 = mode == 1 ? 0 : 1;
      At<WIN> x;
      if (I.open) {
        x = a_cat<WIN>(I, x0, gat<WIN>(I, P, b, r1, i0, n1 - 1, n1));
      } else {
        int j0 = mode == 0 ? n1 - 1 : n1 - 2;
        At<WIN> x2 = mode == 0 ? a_empty<WIN>() : a_node<WIN>(I, arr_new);
        x = a_cat<WIN>(I, a_cat<WIN>(I, x0, gat<WIN>(I, P, b, r1, i0, j0, n1)), x2);
      }
      contrib<WIN>(I, x, dep_new, arr_new, k1, cA);
      for (int f = 0; f < 5; f++) nw[f] = 0.0 + cA[f];
      if (I.nv_on) {
        bool moves_dep = dep_new != m1.y;
        if (moves_dep) fleet_delta = 0.0 + (FL[dep_new].x + FL[m1.y].y);
        fn = !moves_dep;
      }
      break;
    }
  }
  // _old_contrib (batch.py:342-357); closure of the current route from its meta
  const double4 *RC = P.rcon + (size_t)b * P.J;
  double4 o1 = RC[r1];
  double old[5] = {o1.x, o1.y, o1.z, o1.w, (double)m1.w};
  if (two) {
    double4 o2 = RC[r2];
    int4 m2 = RM[r2];
    old[0] = old[0] + o2.x; old[1] = old[1] + o2.y; old[2] = old[2] + o2.z; old[3] = old[3] + o2.w;
    old[4] = old[4] + (double)m2.w;
  }
  Delta D;
  D.dD = nw[0] - old[0];
  D.dV1 = nw[1] - old[1];
  D.dV2 = nw[2] - old[2];
  D.dV3 = nw[3] - old[3];
  D.dV4 = I.theta * ((nw[4] - old[4]) + fleet_delta);
  D.dF = (((D.dD + lam[0] * D.dV1) + lam[1] * D.dV2) + lam[2] * D.dV3) + lam[3] * D.dV4;
  D.fn = fn;
  return D;
}

// table entry without endpoints (read-only in the evaluation kernels)
template <bool WIN>
__device__ __forceinline__ At<WIN> tab_raw(const double *src) {
  const double2 *e = reinterpret_cast<const double2 *>(src);
  At<WIN> a;
  const double2 x = __ldg(e), y = __ldg(e + 1);
  a.dist = x.x; a.load = x.y; a.T = y.x;
  if (WIN) {
    const double2 z = __ldg(e + 2);
    a.E = y.y; a.L = z.x; a.TW = z.y;
  } else {
    a.E = 0.0; a.L = 0.0; a.TW = 0.0;
  }
  a.first = 0; a.last = 0;
  return a;
}

// same-route relocate (OP 0) / swap (OP 1): eval_cand's r1 == r2 branches
// (batch.py:391-463) with every load issued in two waves -- first all that the
// key addresses (route meta and terms, sequence ids, the prefix / segment /
// middle / suffix table entries; an empty middle or suffix reads a harmless
// in-row slot), then the links between the pieces -- instead of one dependent
// load chain per concatenation.  Same pieces, same concatenation order, same
// link values: bit-identical to eval_cand.
template <bool WIN, int OP>
__device__ __forceinline__ Delta eval_intra(const DevInst &I, const DevPop &P, int b, const Cand &c,
                                            const double lam[4]) {
  const int r = c.r1, p1 = c.p1, p2 = c.p2, l1 = c.l1;
  const size_t rb = row_base(P, b, r);
  const int *sq = P.seq + rb;
  const int Kp = P.Kp, FE = P.FE;
  const int4 m1 = P.rmeta[(size_t)b * P.J + r];
  const double4 o1 = P.rcon[(size_t)b * P.J + r];
  // pieces, in concatenation order: X (prefix 0..e), then for relocate
  // [S, M] (before) or [M, S], for swap [B, M, A]; then U (suffix isf..n-1)
  int e, iS, jS, iM, jM, iB = 0, jB = 0, isf;
  bool before = false;
  if (OP == 0) {
    before = p2 <= p1;
    e = before ? p2 : p1;
    iS = p1 + 1; jS = p1 + l1;
    iM = before ? p2 + 1 : p1 + l1 + 1; jM = before ? p1 : p2;
    isf = before ? p1 + l1 + 1 : p2 + 1;
  } else {
    e = p1;
    iS = p1 + 1; jS = p1 + l1;  // segment A
    iB = p2 + 1; jB = p2 + c.l2;
    iM = p1 + l1 + 1; jM = p2;
    isf = p2 + c.l2 + 1;
  }
  const bool midne = jM >= iM;
  const int iM2 = midne ? iM : iS, jM2 = midne ? jM : jS;
  // wave 1
  const int v_e = __ldg(sq + e), v_sf = __ldg(sq + iS), v_sl = __ldg(sq + jS);
  const int v_mf = __ldg(sq + iM2), v_ml = __ldg(sq + jM2), v_uf = __ldg(sq + isf);
  const int v_bf = OP == 1 ? __ldg(sq + iB) : 0, v_bl = OP == 1 ? __ldg(sq + jB) : 0;
  const At<WIN> X = tab_raw<WIN>(P.tabP + (rb + e) * FE);
  const At<WIN> S = tab_raw<WIN>(P.tabT + ((rb + iS) * Kp + jS) * FE);
  const At<WIN> M = tab_raw<WIN>(P.tabT + ((rb + iM2) * Kp + jM2) * FE);
  const At<WIN> U = tab_raw<WIN>(P.tabS + (rb + isf) * FE);
  At<WIN> Bq;
  if (OP == 1) Bq = tab_raw<WIN>(P.tabT + ((rb + iB) * Kp + jB) * FE);
  const int k1 = m1.x, n1 = k1 + (I.open ? 1 : 2);
  const bool sufne = isf <= n1 - 1;
  const int sF = c.rev1 ? v_sl : v_sf, sL = c.rev1 ? v_sf : v_sl;
  // wave 2: the links, in concatenation order
  At<WIN> x;
  if (OP == 0) {
    if (before) {
      const int mlast = midne ? v_ml : sL;
      const Link L1 = link_of(I, v_e, sF);
      const Link L2 = midne ? link_of(I, sL, v_mf) : Link{0.0, 0.0};
      const Link L3 = sufne ? link_of(I, mlast, v_uf) : Link{0.0, 0.0};
      x = a_cat_l<WIN>(X, S, L1);
      if (midne) x = a_cat_l<WIN>(x, M, L2);
      if (sufne) x = a_cat_l<WIN>(x, U, L3);
    } else {
      const int mlast = midne ? v_ml : v_e;
      const Link L1 = midne ? link_of(I, v_e, v_mf) : Link{0.0, 0.0};
      const Link L2 = link_of(I, mlast, sF);
      const Link L3 = sufne ? link_of(I, sL, v_uf) : Link{0.0, 0.0};
      x = X;
      if (midne) x = a_cat_l<WIN>(x, M, L1);
      x = a_cat_l<WIN>(x, S, L2);
      if (sufne) x = a_cat_l<WIN>(x, U, L3);
    }
  } else {
    const int bF = c.rev2 ? v_bl : v_bf, bL = c.rev2 ? v_bf : v_bl;
    const int mlast = midne ? v_ml : bL;
    const Link L1 = link_of(I, v_e, bF);
    const Link L2 = midne ? link_of(I, bL, v_mf) : Link{0.0, 0.0};
    const Link L3 = link_of(I, mlast, sF);
    const Link L4 = sufne ? link_of(I, sL, v_uf) : Link{0.0, 0.0};
    x = a_cat_l<WIN>(X, Bq, L1);
    if (midne) x = a_cat_l<WIN>(x, M, L2);
    x = a_cat_l<WIN>(x, S, L3);
    if (sufne) x = a_cat_l<WIN>(x, U, L4);
  }
  double cA[5];
  contrib<WIN>(I, x, m1.y, m1.z, k1, cA);
  const double old[5] = {o1.x, o1.y, o1.z, o1.w, (double)m1.w};
  Delta D;
  D.dD = (0.0 + cA[0]) - old[0];
  D.dV1 = (0.0 + cA[1]) - old[1];
  D.dV2 = (0.0 + cA[2]) - old[2];
  D.dV3 = (0.0 + cA[3]) - old[3];
  D.dV4 = I.theta * (((0.0 + cA[4]) - old[4]) + 0.0);
  D.dF = (((D.dD + lam[0] * D.dV1) + lam[1] * D.dV2) + lam[2] * D.dV3) + lam[3] * D.dV4;
  D.fn = 1;
  return D;
}

__device__ __forceinline__ bool follower_ok(const Delta &d) {
  return d.dD < -MDR_EPS && fabs(d.dV1) <= MDR_EPS && fabs(d.dV2) <= MDR_EPS && fabs(d.dV3) <= MDR_EPS &&
         fabs(d.dV4) <= MDR_EPS && d.fn;
}

// ---------------------------------------------------------------------------
// implicit enumeration (moves.py:253-464): item index -> candidate, in the
// reference's emission order.  M = current route count of the individual.
// ---------------------------------------------------------------------------
struct EnumDims {
  int M, NC, W, ND, V, nmodes;
};

__device__ __forceinline__ int loc_r(int l) { return l >> 9; }
__device__ __forceinline__ int loc_p(int l) { return l & 511; }

__host__ __device__ __forceinline__ long long op_items(int op, int M, int NC, int W, int ND, int win, int open, int K) {
  long long G = (long long)NC * W;
  switch (op) {
    case 0: return (long long)(win ? 2 : 3) * (G + 2LL * NC * M);
    case 1: return (long long)(win ? 4 : 9) * G;
    case 2: return M < 2 ? 0 : G + 2LL * NC * M + (long long)M * M;
    case 3: return win ? 0 : 2 * G;
    case 4: return (long long)M * K * ND;
    default: return (long long)(open ? 1 : 3) * M * ND;
  }
}

// returns true and fills c if item is a valid candidate
__device__ __forceinline__ bool decode_item(const DevInst &I, const DevPop &P, int b, int op, long long item, int M,
                                            Cand &c) {
  const int *LOC = P.loc + (size_t)b * P.N;
  const int4 *RM = P.rmeta + (size_t)b * P.J;
  const int NC = I.NC, W = I.W, ND = I.ND;
  const long long G = (long long)NC * W;
  c.r2 = -1; c.p2 = -1; c.l1 = 0; c.l2 = 0; c.rev1 = 0; c.rev2 = 0; c.depot = -1; c.mode = -1;
  switch (op) {
    case 0: {  // RELOCATE moves.py:280-311
      long long per = G + 2LL * NC * M;
      int vi = (int)(item / per);
      long long rem = item - (long long)vi * per;
      int len = vi == 0 ? 1 : 2, rev = vi == 2;
      if (rem < G) {
        int u = ND + (int)(rem / W);
        int v = __ldg(I.lists + rem);
        if (v < 0) return false;
        int lu = LOC[u], lv = LOC[v];
        if (lu < 0 || lv < 0) return false;
        int ru = loc_r(lu), pu = loc_p(lu), rv = loc_r(lv), pv = loc_p(lv);
        int ku = RM[ru].x, same = ru == rv, tgt = pv + 1;
        bool ok = (pu + len <= ku) && !(same && tgt > pu && tgt <= pu + len);
        if (!rev) ok = ok && !(same && tgt == pu);
        if (!ok) return false;
        c.r1 = ru; c.p1 = pu; c.r2 = rv; c.p2 = tgt;
      } else {
        rem -= G;
        long long NM = (long long)NC * M;
        int front = rem < NM;
        if (!front) rem -= NM;
        int ub = ND + (int)(rem / M), rb = (int)(rem - (long long)(ub - ND) * M);
        int lub = LOC[ub];
        if (lub < 0) return false;
        int rub = loc_r(lub), pub = loc_p(lub), kub = RM[rub].x;
        int tg = front ? 0 : RM[rb].x, sameb = rub == rb;
        bool ok = (pub + len <= kub) && !(sameb && tg == pub + len);
        if (!rev) ok = ok && !(sameb && tg == pub);
        if (!ok) return false;
        c.r1 = rub; c.p1 = pub; c.r2 = rb; c.p2 = tg;
      }
      c.l1 = len; c.rev1 = rev;
      return true;
    }
    case 1: {  // SWAP moves.py:314-358
      int ci = (int)(item / G);
      long long rem = item - (long long)ci * G;
      int lu, lv, au, av;
      if (!I.win) {
        // (lu,lv,au,av) in the order of moves.py:326-329
        const int T[9] = {0x1100, 0x1200, 0x1201, 0x2100, 0x2110, 0x2200, 0x2201, 0x2210, 0x2211};
        int t = T[ci];
        lu = (t >> 12) & 0xf; lv = (t >> 8) & 0xf; au = (t >> 4) & 0xf; av = t & 0xf;
      } else {
        lu = ci < 2 ? 1 : 2; lv = (ci & 1) ? 2 : 1; au = 0; av = 0;
      }
      int u = ND + (int)(rem / W);
      int v = __ldg(I.lists + rem);
      if (v < 0 || v == u) return false;
      int Lu = LOC[u], Lv = LOC[v];
      if (Lu < 0 || Lv < 0) return false;
      int ru = loc_r(Lu), pu = loc_p(Lu), rv = loc_r(Lv), pv = loc_p(Lv);
      int same = ru == rv, flip = same && pu > pv;
      int q1 = flip ? pv : pu, q2 = flip ? pu : pv;
      int l1 = flip ? lv : lu, l2 = flip ? lu : lv;
      int b1 = flip ? av : au, b2 = flip ? au : av;
      bool fits = (q1 + l1 <= RM[ru].x) && (q2 + l2 <= RM[rv].x);
      if (!(fits && (!same || q2 >= q1 + l1))) return false;
      c.r1 = ru; c.p1 = q1; c.r2 = rv; c.p2 = q2; c.l1 = l1; c.l2 = l2; c.rev1 = b1; c.rev2 = b2;
      return true;
    }
    case 3: {  // TWO_OPT moves.py:361-372
      int dir = item >= G;
      long long rem = dir ? item - G : item;
      int u = ND + (int)(rem / W);
      int v = __ldg(I.lists + rem);
      if (v < 0) return false;
      int Lu = LOC[u], Lv = LOC[v];
      if (Lu < 0 || Lv < 0) return false;
      int ru = loc_r(Lu), pu = loc_p(Lu), rv = loc_r(Lv), pv = loc_p(Lv);
      if (ru != rv) return false;
      if (dir == 0) { if (!(pv >= pu + 2)) return false; c.p1 = pu + 1; c.p2 = pv; }
      else { if (!(pu >= pv + 2)) return false; c.p1 = pv + 1; c.p2 = pu; }
      c.r1 = ru;
      return true;
    }
    case 2: {  // TWO_OPT_STAR moves.py:375-405
      if (item < G) {
        int v = __ldg(I.lists + item);
        int u = ND + (int)(item / W);
        if (v < 0) return false;
        int Lu = LOC[u], Lv = LOC[v];
        if (Lu < 0 || Lv < 0) return false;
        int ru = loc_r(Lu), rv = loc_r(Lv);
        if (ru == rv) return false;
        c.r1 = ru; c.p1 = loc_p(Lu) + 1; c.r2 = rv; c.p2 = loc_p(Lv);
        return true;
      }
      long long rem = item - G;
      long long NM = (long long)NC * M;
      if (rem < 2 * NM) {
        int fam = rem >= NM;
        if (fam) rem -= NM;
        int ub = ND + (int)(rem / M), rb = (int)(rem - (long long)(ub - ND) * M);
        int lub = LOC[ub];
        if (lub < 0) return false;
        int rub = loc_r(lub), pub = loc_p(lub);
        if (rub == rb) return false;
        if (fam == 0) {
          int q1 = pub + 1, q2 = RM[rb].x;
          bool drop = (q1 == RM[rub].x);
          if (!I.open) drop = drop && (RM[rub].z == RM[rb].z);
          if (drop) return false;
          c.r1 = rub; c.p1 = q1; c.r2 = rb; c.p2 = q2;
        } else {
          c.r1 = rb; c.p1 = 0; c.r2 = rub; c.p2 = pub;
        }
        return true;
      }
      rem -= 2 * NM;
      int ra = (int)(rem / M), rb = (int)(rem - (long long)ra * M);
      if (ra == rb) return false;
      c.r1 = ra; c.p1 = 0; c.r2 = rb; c.p2 = RM[rb].x;
      return true;
    }
    case 4: {  // DEPOT_INSERT moves.py:408-422
      int d = (int)(item % ND);
      long long rp = item / ND;
      int r = (int)(rp / P.K), p = (int)(rp - (long long)r * P.K);
      int4 mr = RM[r];
      if (p >= mr.x) return false;
      bool closes_same = I.open || mr.z == mr.y;
      if (p == 0 && d == mr.y && closes_same) return false;
      c.r1 = r; c.p1 = p; c.depot = d;
      return true;
    }
    default: {  // DEPOT_REPLACE moves.py:425-441
      long long MD = (long long)M * ND;
      int mode = (int)(item / MD);
      long long rem = item - (long long)mode * MD;
      int r = (int)(rem / ND), d = (int)(rem - (long long)r * ND);
      int4 mr = RM[r];
      bool ok = mode == 0 ? d != mr.y : (mode == 1 ? d != mr.z : !(d == mr.y && d == mr.z));
      if (!ok) return false;
      c.r1 = r; c.p1 = 0; c.depot = d; c.mode = mode;
      return true;
    }
  }
}

}  // namespace mdr
