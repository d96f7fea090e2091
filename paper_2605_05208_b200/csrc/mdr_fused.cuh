// mdr_fused.cuh -- warp-per-task fused enumerate + evaluate + reduce.
//
// A round's work list is flattened into tasks: for relocate / swap / 2-opt /
// 2-opt* one task per customer u of an individual (its granular and boundary
// targets, moves.py:253-405), plus one task per route for the 2-opt* route
// pairs and the depot operators.  One warp owns a task: everything that
// depends only on u (route, position, removal terms, u's segments) is
// computed once per warp; the 32 lanes sweep the targets.  No block barrier:
// each warp writes one (ord(dF), key) partial and a candidate count per task,
// and appends followers with warp-aggregated atomics.
//
// Every candidate goes through the same fp64 expression DAG as
// batch.evaluate_candidates (see eval_cand in mdr_device.cuh); rare intra-route
// candidates call eval_cand itself.
#pragma once
#include "mdr_device.cuh"

namespace mdr {

// per-individual base pointers (warp-uniform)
struct IV {
  const int *seq;
  const double *tP, *tS;
  const int4 *rm;
  const double4 *rc;
  const int *loc, *nxs;
  const double2 *fl;
  int Kp, M;
};

__device__ __forceinline__ double4 ldg4(const double4 *p) {
  const double2 *q = reinterpret_cast<const double2 *>(p);
  double2 a = __ldg(q), b = __ldg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

template <bool WIN>
struct FE_ {
  static constexpr int v = WIN ? 6 : 4;
};

__device__ __forceinline__ IV make_iv(const DevPop &P, int b) {
  IV v;
  size_t rows = (size_t)b * P.J;
  v.seq = P.seq + rows * P.Kp;
  v.tP = P.tabP + rows * P.Kp * P.FE;
  v.tS = P.tabS + rows * P.Kp * P.FE;
  v.rm = P.rmeta + rows;
  v.rc = P.rcon + rows;
  v.loc = P.loc + (size_t)b * P.N;
  v.nxs = P.nxs + (size_t)b * P.N;
  v.fl = P.fleet + (size_t)b * P.ND;
  v.Kp = P.Kp;
  v.M = P.m[b];
  return v;
}

template <bool WIN>
__device__ __forceinline__ At<WIN> ld_tab(const double *tab, int off) {
  const double2 *e = reinterpret_cast<const double2 *>(tab + off * FE_<WIN>::v);
  At<WIN> a;
  double2 x = __ldg(e), y = __ldg(e + 1);
  a.dist = x.x; a.load = x.y; a.T = y.x;
  if (WIN) {
    double2 z = __ldg(e + 2);
    a.E = y.y; a.L = z.x; a.TW = z.y;
  } else {
    a.E = 0.0; a.L = 0.0; a.TW = 0.0;
  }
  return a;
}

// prefix (0..j) of route r
template <bool WIN>
__device__ __forceinline__ At<WIN> pre(const IV &v, int r, int j) {
  At<WIN> a = ld_tab<WIN>(v.tP, r * v.Kp + j);
  const int *sq = v.seq + r * v.Kp;
  a.first = __ldg(sq);
  a.last = __ldg(sq + j);
  return a;
}

// suffix (i..n-1) of route r, empty when i > n-1
template <bool WIN>
__device__ __forceinline__ At<WIN> suf(const IV &v, int r, int i, int n) {
  if (i > n - 1) return a_empty<WIN>();
  At<WIN> a = ld_tab<WIN>(v.tS, r * v.Kp + i);
  const int *sq = v.seq + r * v.Kp;
  a.first = __ldg(sq + i);
  a.last = __ldg(sq + n - 1);
  return a;
}

// _route_penalties with exact-zero short cuts (0/Q is +0 exactly)
template <bool WIN>
__device__ __forceinline__ void contrib_fast(const DevInst &I, const At<WIN> &a, int dep, int arr, int kc, double o[5]) {
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

struct Acc {  // lane-local running leader + candidate count
  unsigned long long o, k;
  int n;
};

__device__ __forceinline__ void finish_delta(const DevInst &I, const double nw[5], const double old[5], double fleet_delta,
                                             const double lam[4], Delta &D) {
  D.dD = nw[0] - old[0];
  D.dV1 = nw[1] - old[1];
  D.dV2 = nw[2] - old[2];
  D.dV3 = nw[3] - old[3];
  D.dV4 = I.theta * ((nw[4] - old[4]) + fleet_delta);
  D.dF = (((D.dD + lam[0] * D.dV1) + lam[1] * D.dV2) + lam[2] * D.dV3) + lam[3] * D.dV4;
}

// record one evaluated candidate (lane-local) and report whether it is a follower
__device__ __forceinline__ bool record(Acc &acc, const Delta &D, unsigned long long key, bool mm, int *nanflag) {
  acc.n++;
  if (D.dF != D.dF) {
    atomicOr(nanflag, 1);
    return false;
  }
  unsigned long long o = ord_of(D.dF);
  if (o < acc.o || (o == acc.o && key < acc.k)) { acc.o = o; acc.k = key; }
  return mm && follower_ok(D);
}

// warp-aggregated follower append (full-warp call)
__device__ __forceinline__ void append_fol(const DevPop &P, int b, bool fol, unsigned long long o, unsigned long long k) {
  unsigned fm = __ballot_sync(0xffffffffu, fol);
  if (!fm) return;
  int lane = threadIdx.x & 31;
  int leader = __ffs(fm) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(&P.fcount[b], __popc(fm));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (fol) {
    int at = base + __popc(fm & ((1u << lane) - 1));
    if (at < P.Fcap) P.fol[(size_t)b * P.Fcap + at] = make_ulonglong2(o, k);
  }
}

__device__ __forceinline__ unsigned long long key_of(int r1, int p1, int r2, int p2, int l1, int l2, int v1, int v2,
                                                     int depot, int mode) {
  Cand c;
  c.r1 = r1; c.p1 = p1; c.r2 = r2; c.p2 = p2; c.l1 = l1; c.l2 = l2; c.rev1 = v1; c.rev2 = v2; c.depot = depot;
  c.mode = mode;
  return pack_key(c);
}

// queue a candidate for the generic evaluator (k_eval_g); full-warp call
__device__ __forceinline__ void enqueue_g(const DevPop &P, int b, int op, bool q, unsigned long long key) {
  unsigned qm = __ballot_sync(0xffffffffu, q);
  if (!qm) return;
  const int region = P.gbase[1] > 0 ? (op >= 3 ? 0 : (op == 0 ? 1 : 2)) : 1;  // see DevPop::gq
  const int cap = P.gbase[region + 1] - P.gbase[region];
  ulonglong2 *Q = P.gq + P.gbase[region];
  int lane = threadIdx.x & 31;
  int leader = __ffs(qm) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(P.gcount + region, __popc(qm));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (q) {
    int at = base + __popc(qm & ((1u << lane) - 1));
    if (at < cap) Q[at] = make_ulonglong2(key, (unsigned long long)(b | (op << 24)));
  }
}

// 128-bit min of {ord(dF), key} into the individual's leader slot
__device__ __forceinline__ void leader_min(ulonglong2 *addr, unsigned long long o, unsigned long long k) {
  if (o == ~0ull) return;
  const volatile unsigned long long *va = reinterpret_cast<const volatile unsigned long long *>(addr);
  ulonglong2 cur;
  cur.x = va[0];
  cur.y = va[1];
  while (o < cur.x || (o == cur.x && k < cur.y)) {
    ulonglong2 prev = atomicCAS(addr, cur, make_ulonglong2(o, k));
    if (prev.x == cur.x && prev.y == cur.y) break;
    cur = prev;
  }
}

// per-warp shared-memory staging of warp-uniform (u-side) attributes
template <bool WIN>
__device__ __forceinline__ void st_at(double *U, const At<WIN> &a) {
  U[0] = a.dist; U[1] = a.load; U[2] = a.T;
  if (WIN) { U[3] = a.E; U[4] = a.L; U[5] = a.TW; }
}
template <bool WIN>
__device__ __forceinline__ At<WIN> ld_at(const double *U, int first, int last) {
  At<WIN> a;
  a.dist = U[0]; a.load = U[1]; a.T = U[2];
  if (WIN) { a.E = U[3]; a.L = U[4]; a.TW = U[5]; }
  else { a.E = 0.0; a.L = 0.0; a.TW = 0.0; }
  a.first = first; a.last = last;
  return a;
}
#define MDR_USLOT 32  // doubles of per-warp staging

// ---------------------------------------------------------------------------
// RELOCATE, task = customer u (moves.py:280-311, batch.py:391-428)
// ---------------------------------------------------------------------------
template <bool WIN>
__device__ void task_relocate(const DevInst &I, const DevPop &P, const IV &v, int b, int u, const double lam[4],
                              bool mm, Acc &acc, double *U) {
  const int lane = threadIdx.x & 31;
  const int lu = __ldg(v.loc + u);
  if (lu < 0) return;
  const int ru = loc_r(lu), pu = loc_p(lu);
  const int4 m1 = __ldg(v.rm + ru);
  const int k1 = m1.x;
  const int nxt = pu + 2 <= k1 ? __ldg(v.seq + ru * v.Kp + pu + 2) : u;
  // u-side terms, once per warp (lane 0), staged in shared memory:
  // U[0..4] removal contribution l=1, U[5..9] l=2, U[10..15] seg l=1, U[16..21] seg l=2,
  // U[22..25] old route terms of ru, U[26] fleet_dec of ru's depot
  if (lane == 0) {
    const int n1 = k1 + (I.open ? 1 : 2);
    At<WIN> P1 = pre<WIN>(v, ru, pu);
    for (int l = 1; l <= 2; l++) {
      if (pu + l <= k1) {
        At<WIN> A = a_cat<WIN>(I, P1, suf<WIN>(v, ru, pu + l + 1, n1));
        contrib_fast<WIN>(I, A, m1.y, m1.z, k1 - l, U + 5 * (l - 1));
      }
    }
    At<WIN> s1 = a_node<WIN>(I, u);
    st_at<WIN>(U + 10, s1);
    if (pu + 2 <= k1) st_at<WIN>(U + 16, a_cat_ne<WIN>(I, s1, a_node<WIN>(I, nxt)));
    double4 rc1 = ldg4(v.rc + ru);
    U[22] = rc1.x; U[23] = rc1.y; U[24] = rc1.z; U[25] = rc1.w;
    U[26] = I.nv_on ? __ldg(v.fl + m1.y).y : 0.0;
  }
  __syncwarp();
  const int nvar = I.win ? 2 : 3;
  const int W = I.W;
  const int T = W + 2 * v.M;
  const int *lst = I.lists + (size_t)(u - I.ND) * W;
  for (int base = 0; base < T; base += 32) {
    const int t = base + lane;
    int rv = -1, tgt = -1;
    const bool gran = t < W;
    if (t < W) {
      int vv = __ldg(lst + t);
      if (vv >= 0) {
        int lv = __ldg(v.loc + vv);
        if (lv >= 0) { rv = loc_r(lv); tgt = loc_p(lv) + 1; }
      }
    } else if (t < T) {
      int tb = t - W;
      bool front = tb < v.M;
      rv = front ? tb : tb - v.M;
      tgt = front ? 0 : __ldg(v.rm + rv).x;
    }
    const bool same = rv == ru;
    bool loaded = false;
    At<WIN> P2, S2;
    int4 m2;
    for (int vi = 0; vi < nvar; vi++) {
      const int len = vi == 0 ? 1 : 2, rev = vi == 2;
      bool ok = rv >= 0 && pu + len <= k1;
      if (gran) ok = ok && !(same && tgt > pu && tgt <= pu + len);
      else ok = ok && !(same && tgt == pu + len);
      if (!rev) ok = ok && !(same && tgt == pu);
      bool fol = false, gqf = false;
      unsigned long long o = 0, key = 0;
      if (ok) {
        key = key_of(ru, pu, rv, tgt, len, 0, rev, 0, -1, -1);
        if (same) {
          gqf = true;
        } else {
          if (!loaded) {
            m2 = __ldg(v.rm + rv);
            P2 = pre<WIN>(v, rv, tgt);
            S2 = suf<WIN>(v, rv, tgt + 1, m2.x + (I.open ? 1 : 2));
            loaded = true;
          }
          At<WIN> seg = ld_at<WIN>(U + (len == 1 ? 10 : 16), rev ? (len == 1 ? u : nxt) : u,
                                   rev ? u : (len == 1 ? u : nxt));
          At<WIN> B = a_cat_ne<WIN>(I, P2, seg);
          if (S2.first >= 0) B = a_cat_ne<WIN>(I, B, S2);
          double cB[5], nw[5];
          contrib_fast<WIN>(I, B, m2.y, m2.z, m2.x + len, cB);
          const double *ca = U + 5 * (len - 1);
#pragma unroll
          for (int f = 0; f < 5; f++) nw[f] = (0.0 + ca[f]) + cB[f];
          double fleet_delta = 0.0;
          int fn = 1;
          if (I.nv_on && k1 - len == 0) { fleet_delta = 0.0 + U[26]; fn = 0; }
          const double4 rc2 = ldg4(v.rc + rv);
          double old[5] = {U[22] + rc2.x, U[23] + rc2.y, U[24] + rc2.z, U[25] + rc2.w, (double)m1.w + (double)m2.w};
          Delta D;
          finish_delta(I, nw, old, fleet_delta, lam, D);
          D.fn = fn;
          fol = record(acc, D, key, mm, P.nanflag + b);
          o = ord_of(D.dF);
        }
      }
      append_fol(P, b, fol, o, key);
      enqueue_g(P, b, 0, gqf, key);
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// SWAP, task = customer u (moves.py:314-358, batch.py:430-463)
// ---------------------------------------------------------------------------
template <bool WIN>
__device__ void task_swap(const DevInst &I, const DevPop &P, const IV &v, int b, int u, const double lam[4], bool mm,
                          Acc &acc, double *U) {
  const int lane = threadIdx.x & 31;
  const int lu = __ldg(v.loc + u);
  if (lu < 0) return;
  const int ru = loc_r(lu), pu = loc_p(lu);
  const int4 m1 = __ldg(v.rm + ru);
  const int k1 = m1.x, n1 = k1 + (I.open ? 1 : 2);
  const int nxtu = pu + 2 <= k1 ? __ldg(v.seq + ru * v.Kp + pu + 2) : u;
  const int dep1 = __ldg(v.seq + ru * v.Kp), lastP1 = __ldg(v.seq + ru * v.Kp + pu);
  // U[0..5] seg u l=1, U[6..11] seg u l=2, U[12..17] prefix (0..pu), U[18..21] old terms of ru
  if (lane == 0) {
    At<WIN> s1 = a_node<WIN>(I, u);
    st_at<WIN>(U, s1);
    if (pu + 2 <= k1) st_at<WIN>(U + 6, a_cat_ne<WIN>(I, s1, a_node<WIN>(I, nxtu)));
    st_at<WIN>(U + 12, pre<WIN>(v, ru, pu));
    double4 rc1 = ldg4(v.rc + ru);
    U[18] = rc1.x; U[19] = rc1.y; U[20] = rc1.z; U[21] = rc1.w;
  }
  __syncwarp();
  const int W = I.W;
  const int *lst = I.lists + (size_t)(u - I.ND) * W;
  for (int base = 0; base < W; base += 32) {
    const int t = base + lane;
    int vv = t < W ? __ldg(lst + t) : -1;
    int rv = -1, pv = -1;
    if (vv >= 0 && vv != u) {
      int lv = __ldg(v.loc + vv);
      if (lv >= 0) { rv = loc_r(lv); pv = loc_p(lv); }
    }
    const bool same = rv == ru;
    int4 m2 = make_int4(0, 0, 0, 0);
    At<WIN> P2;
    int nxtv = vv;
    if (rv >= 0 && !same) {
      m2 = __ldg(v.rm + rv);
      P2 = pre<WIN>(v, rv, pv);
      if (pv + 2 <= m2.x) nxtv = __ldg(v.seq + rv * v.Kp + pv + 2);
    }
    // combos grouped by lv so one segment of v is live at a time (order is irrelevant:
    // every candidate is scored independently)
    for (int lv_ = 1; lv_ <= 2; lv_++) {
      At<WIN> segB;
      if (rv >= 0 && !same && pv + lv_ <= m2.x) {
        segB = a_node<WIN>(I, vv);
        if (lv_ == 2) segB = a_cat_ne<WIN>(I, segB, a_node<WIN>(I, nxtv));
      }
      const int ncomb = I.win ? 2 : (lv_ == 1 ? 3 : 6);
      for (int ci = 0; ci < ncomb; ci++) {
        // (lu, au, av) for this lv (moves.py:325-332)
        int lu_, au, av;
        if (I.win) { lu_ = ci + 1; au = 0; av = 0; }
        else if (lv_ == 1) { lu_ = ci == 0 ? 1 : 2; au = ci == 2; av = 0; }
        else { lu_ = ci < 2 ? 1 : 2; av = ci & 1; au = ci >= 4; }
        bool fol = false, gqf = false;
        unsigned long long o = 0, key = 0;
        if (rv >= 0) {
          if (same) {
            int flip = pu > pv;
            Cand c;
            c.r1 = ru; c.r2 = rv;
            c.p1 = flip ? pv : pu; c.p2 = flip ? pu : pv;
            c.l1 = flip ? lv_ : lu_; c.l2 = flip ? lu_ : lv_;
            c.rev1 = flip ? av : au; c.rev2 = flip ? au : av;
            c.depot = -1; c.mode = -1;
            gqf = (c.p1 + c.l1 <= k1) && (c.p2 + c.l2 <= k1) && (c.p2 >= c.p1 + c.l1);
            key = pack_key(c);
          } else if (pu + lu_ <= k1 && pv + lv_ <= m2.x) {
            const int k2 = m2.x, n2 = k2 + (I.open ? 1 : 2);
            const int ua = lu_ == 1 ? u : nxtu;
            At<WIN> sA = ld_at<WIN>(U + (lu_ == 1 ? 0 : 6), au ? ua : u, au ? u : ua);
            At<WIN> sB = segB;
            if (av) swap_ends(sB);
            At<WIN> A = a_cat_ne<WIN>(I, ld_at<WIN>(U + 12, dep1, lastP1), sB);
            if (pu + lu_ + 1 <= n1 - 1) A = a_cat_ne<WIN>(I, A, suf<WIN>(v, ru, pu + lu_ + 1, n1));
            double cA[5], cB[5], nw[5];
            contrib_fast<WIN>(I, A, m1.y, m1.z, k1 - lu_ + lv_, cA);
            At<WIN> B = a_cat_ne<WIN>(I, P2, sA);
            if (pv + lv_ + 1 <= n2 - 1) B = a_cat_ne<WIN>(I, B, suf<WIN>(v, rv, pv + lv_ + 1, n2));
            contrib_fast<WIN>(I, B, m2.y, m2.z, k2 - lv_ + lu_, cB);
#pragma unroll
            for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
            const double4 rc2 = ldg4(v.rc + rv);
            double old[5] = {U[18] + rc2.x, U[19] + rc2.y, U[20] + rc2.z, U[21] + rc2.w, (double)m1.w + (double)m2.w};
            Delta D;
            finish_delta(I, nw, old, 0.0, lam, D);
            D.fn = 1;
            key = key_of(ru, pu, rv, pv, lu_, lv_, au, av, -1, -1);
            fol = record(acc, D, key, mm, P.nanflag + b);
            o = ord_of(D.dF);
          }
        }
        append_fol(P, b, fol, o, key);
        enqueue_g(P, b, 1, gqf, key);
      }
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// TWO_OPT, task = customer u (moves.py:361-372); symmetric variants only
// ---------------------------------------------------------------------------
template <bool WIN>
__device__ void task_two_opt(const DevInst &I, const DevPop &P, const IV &v, int b, int u, const double lam[4],
                             bool mm, Acc &acc) {
  const int lane = threadIdx.x & 31;
  const int lu = __ldg(v.loc + u);
  if (lu < 0) return;
  const int ru = loc_r(lu), pu = loc_p(lu);
  const int W = I.W;
  const int *lst = I.lists + (size_t)(u - I.ND) * W;
  for (int base = 0; base < W; base += 32) {
    const int t = base + lane;
    int vv = t < W ? __ldg(lst + t) : -1;
    bool gqf = false;
    unsigned long long key = 0;
    if (vv >= 0) {
      int lv = __ldg(v.loc + vv);
      if (lv >= 0 && loc_r(lv) == ru) {
        int pv = loc_p(lv);
        // the fwd (pv >= pu+2) and bwd (pu >= pv+2) families are disjoint
        if (pv >= pu + 2) { gqf = true; key = key_of(ru, pu + 1, -1, pv, 0, 0, 0, 0, -1, -1); }
        else if (pu >= pv + 2) { gqf = true; key = key_of(ru, pv + 1, -1, pu, 0, 0, 0, 0, -1, -1); }
      }
    }
    enqueue_g(P, b, 3, gqf, key);
  }
}

// 2-opt* evaluation of (r1, p1, r2, p2) (batch.py:475-494)
template <bool WIN>
__device__ __forceinline__ bool eval_tos(const DevInst &I, const DevPop &P, const IV &v, int b, int r1, int p1, int r2,
                                         int p2, const double lam[4], Acc &acc, bool mm, unsigned long long &o,
                                         unsigned long long &key) {
  const int4 m1 = __ldg(v.rm + r1), m2 = __ldg(v.rm + r2);
  const int k1 = m1.x, k2 = m2.x;
  const int n1 = k1 + (I.open ? 1 : 2), n2 = k2 + (I.open ? 1 : 2);
  At<WIN> A = pre<WIN>(v, r1, p1);
  if (p2 + 1 <= n2 - 1) A = a_cat_ne<WIN>(I, A, suf<WIN>(v, r2, p2 + 1, n2));
  At<WIN> B = pre<WIN>(v, r2, p2);
  if (p1 + 1 <= n1 - 1) B = a_cat_ne<WIN>(I, B, suf<WIN>(v, r1, p1 + 1, n1));
  const int kA = p1 + (k2 - p2), kB = p2 + (k1 - p1);
  double cA[5], cB[5], nw[5];
  contrib_fast<WIN>(I, A, m1.y, m2.z, kA, cA);
  contrib_fast<WIN>(I, B, m2.y, m1.z, kB, cB);
#pragma unroll
  for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
  double fleet_delta = 0.0;
  int fn = 1;
  if (I.nv_on) {
    fleet_delta = (0.0 + (kA == 0 ? __ldg(v.fl + m1.y).y : 0.0)) + (kB == 0 ? __ldg(v.fl + m2.y).y : 0.0);
    fn = (kA > 0) && (kB > 0);
  }
  const double4 rc1 = ldg4(v.rc + r1), rc2 = ldg4(v.rc + r2);
  double old[5] = {rc1.x + rc2.x, rc1.y + rc2.y, rc1.z + rc2.z, rc1.w + rc2.w, (double)m1.w + (double)m2.w};
  Delta D;
  finish_delta(I, nw, old, fleet_delta, lam, D);
  D.fn = fn;
  key = key_of(r1, p1, r2, p2, 0, 0, 0, 0, -1, -1);
  bool f = record(acc, D, key, mm, P.nanflag + b);
  o = ord_of(D.dF);
  return f;
}

// TWO_OPT_STAR, task = customer u: granular cut + the two boundary families (moves.py:375-400)
template <bool WIN>
__device__ void task_tos_u(const DevInst &I, const DevPop &P, const IV &v, int b, int u, const double lam[4], bool mm,
                           Acc &acc) {
  const int lane = threadIdx.x & 31;
  const int lu = __ldg(v.loc + u);
  if (lu < 0) return;
  const int ru = loc_r(lu), pu = loc_p(lu);
  const int4 mu = __ldg(v.rm + ru);
  const int W = I.W, M = v.M;
  const int T = W + 2 * M;
  const int *lst = I.lists + (size_t)(u - I.ND) * W;
  for (int base = 0; base < T; base += 32) {
    const int t = base + lane;
    int r1 = -1, p1 = 0, r2 = 0, p2 = 0;
    if (t < W) {
      int vv = __ldg(lst + t);
      if (vv >= 0) {
        int lv = __ldg(v.loc + vv);
        if (lv >= 0 && loc_r(lv) != ru) { r1 = ru; p1 = pu + 1; r2 = loc_r(lv); p2 = loc_p(lv); }
      }
    } else if (t < W + M) {
      int rb = t - W;
      if (rb != ru) {
        int4 mb = __ldg(v.rm + rb);
        bool drop = (pu + 1 == mu.x);
        if (!I.open) drop = drop && (mu.z == mb.z);
        if (!drop) { r1 = ru; p1 = pu + 1; r2 = rb; p2 = mb.x; }
      }
    } else if (t < T) {
      int rb = t - W - M;
      if (rb != ru) { r1 = rb; p1 = 0; r2 = ru; p2 = pu; }
    }
    bool fol = false;
    unsigned long long o = 0, key = 0;
    if (r1 >= 0) fol = eval_tos<WIN>(I, P, v, b, r1, p1, r2, p2, lam, acc, mm, o, key);
    append_fol(P, b, fol, o, key);
  }
}

// TWO_OPT_STAR route pairs (ra, 0, rb, k_rb), task = route ra (moves.py:401-404)
template <bool WIN>
__device__ void task_tos_r(const DevInst &I, const DevPop &P, const IV &v, int b, int ra, const double lam[4], bool mm,
                           Acc &acc) {
  const int lane = threadIdx.x & 31;
  for (int base = 0; base < v.M; base += 32) {
    const int rb = base + lane;
    bool fol = false;
    unsigned long long o = 0, key = 0;
    if (rb < v.M && rb != ra) fol = eval_tos<WIN>(I, P, v, b, ra, 0, rb, __ldg(v.rm + rb).x, lam, acc, mm, o, key);
    append_fol(P, b, fol, o, key);
  }
}

// DEPOT_INSERT, task = route r: lanes over (p, d) (moves.py:408-422)
template <bool WIN>
__device__ void task_di(const DevInst &I, const DevPop &P, const IV &v, int b, int r, const double lam[4], bool mm,
                        Acc &acc) {
  const int lane = threadIdx.x & 31;
  const int4 mr = __ldg(v.rm + r);
  const int T = mr.x * I.ND;
  const bool closes_same = I.open || mr.z == mr.y;
  for (int base = 0; base < T; base += 32) {
    const int t = base + lane;
    bool gqf = false;
    unsigned long long key = 0;
    if (t < T) {
      int p = t / I.ND, d = t - p * I.ND;
      if (!(p == 0 && d == mr.y && closes_same)) { gqf = true; key = key_of(r, p, -1, -1, 0, 0, 0, 0, d, -1); }
    }
    enqueue_g(P, b, 4, gqf, key);
  }
}

// DEPOT_REPLACE, task = route r: lanes over (mode, d) (moves.py:425-441)
template <bool WIN>
__device__ void task_dr(const DevInst &I, const DevPop &P, const IV &v, int b, int r, const double lam[4], bool mm,
                        Acc &acc) {
  const int lane = threadIdx.x & 31;
  const int4 mr = __ldg(v.rm + r);
  const int nm = I.open ? 1 : 3;
  const int T = nm * I.ND;
  for (int base = 0; base < T; base += 32) {
    const int t = base + lane;
    bool gqf = false;
    unsigned long long key = 0;
    if (t < T) {
      int mode = t / I.ND, d = t - mode * I.ND;
      bool ok = mode == 0 ? d != mr.y : (mode == 1 ? d != mr.z : !(d == mr.y && d == mr.z));
      if (ok) { gqf = true; key = key_of(r, 0, -1, -1, 0, 0, 0, 0, d, mode); }
    }
    enqueue_g(P, b, 5, gqf, key);
  }
}

// tasks of one individual for operator op
__host__ __device__ __forceinline__ int op_tasks(int op, int M, int NC, int win) {
  switch (op) {
    case 0: case 1: return NC;
    case 2: return M < 2 ? 0 : NC + M;
    case 3: return win ? 0 : NC;
    default: return M;
  }
}

}  // namespace mdr
