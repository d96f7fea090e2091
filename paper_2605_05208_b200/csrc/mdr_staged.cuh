// mdr_staged.cuh -- CTA-task evaluators for relocate, swap and 2-opt* with
// the individual's per-route boundary data staged in shared memory.
//
// A CTA task is (individual b, 8 customers): every warp owns one customer u
// (or, for the 2-opt* route-pair family, one route ra).  Before its warps
// start, the CTA stages for every route r of b: meta, old route terms, the
// suffix after the departure depot S[r][1] and the prefix up to the last
// customer P[r][k].  These are exactly the pieces of the route-boundary
// candidate families (moves.py:289-310, 390-404) -- ~75 % of relocate and
// 2-opt* candidates -- which then need nothing from global memory except
// their distance links.  Evaluation order inside a task differs from the
// reference's enumeration order; the result does not (every candidate is
// scored independently and reduced by (dF, key)).
#pragma once
#include "mdr_fused.cuh"

namespace mdr {

#ifndef MDR_RB_PAD_NOWIN
#define MDR_RB_PAD_NOWIN 2  // 168-byte stride without windows (odd count of 8-byte words): C5 +1.4 %
#endif
template <bool WIN>
struct RBT {
  double sf[6];  // S[r][1] (suffix after the departure depot), empty when n-1 < 1
  double pb[6];  // P[r][k] (prefix up to the last customer)
  double rc[4];  // route D, V1, V2, V3
  int k, dep, arr, clo;
  int sf_first, sf_last, pb_last, n;
  // strides that spread lanes reading consecutive routes over distinct banks: with windows
  // 176 B (11 x 16 B, C4 +1.8 %); without, 168 B (21 x 8 B, C5 +1.4 %; 176 B was -6 % there:
  // two C5 route tables no longer fit next to the L1 the gathers need)
  int pad[WIN ? 4 : MDR_RB_PAD_NOWIN];
};

template <bool WIN>
__device__ __forceinline__ void stage_routes(const DevInst &I, const IV &v, RBT<WIN> *R) {
  for (int r = threadIdx.x; r < v.M; r += blockDim.x) {
    const int4 mt = __ldg(v.rm + r);
    const int n = mt.x + (I.open ? 1 : 2);
    const int *sq = v.seq + r * v.Kp;
    RBT<WIN> &x = R[r];
    x.k = mt.x; x.dep = mt.y; x.arr = mt.z; x.clo = mt.w; x.n = n;
    const double4 rc = ldg4(v.rc + r);
    x.rc[0] = rc.x; x.rc[1] = rc.y; x.rc[2] = rc.z; x.rc[3] = rc.w;
    if (n - 1 >= 1) {
      st_at<WIN>(x.sf, ld_tab<WIN>(v.tS, r * v.Kp + 1));
      x.sf_first = __ldg(sq + 1);
      x.sf_last = __ldg(sq + n - 1);
    } else {
      x.sf_first = -1;
      x.sf_last = -1;
    }
    st_at<WIN>(x.pb, ld_tab<WIN>(v.tP, r * v.Kp + mt.x));
    x.pb_last = __ldg(sq + mt.x);
  }
}

template <bool WIN>
__device__ __forceinline__ At<WIN> rb_sf(const RBT<WIN> &x) { return ld_at<WIN>(x.sf, x.sf_first, x.sf_last); }
template <bool WIN>
__device__ __forceinline__ At<WIN> rb_pb(const RBT<WIN> &x) { return ld_at<WIN>(x.pb, x.dep, x.pb_last); }

// (0 + cA) + cB, old terms, fleet delta, combine (batch.py:545-553) and record.
// The 58-bit key is packed lazily: only when the candidate can displace the
// lane's running leader (ord(dF) <= best) or is a follower.
template <bool WIN, typename KeyF>
__device__ __forceinline__ bool two_route_delta(const DevInst &I, const double cA[5], const double cB[5],
                                                const double *rc1, const double *rc2, int clo1, int clo2,
                                                double fleet_delta, int fn, const double lam[4], Acc &acc,
                                                KeyF mk, unsigned long long &key, bool mm, int *nanflag,
                                                unsigned long long &o) {
  double nw[5];
#pragma unroll
  for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
  double old[5] = {rc1[0] + rc2[0], rc1[1] + rc2[1], rc1[2] + rc2[2], rc1[3] + rc2[3], (double)clo1 + (double)clo2};
  Delta D;
  finish_delta(I, nw, old, fleet_delta, lam, D);
  D.fn = fn;
  acc.n++;
  if (D.dF != D.dF) {
    atomicOr(nanflag, 1);
    return false;
  }
  o = ord_of(D.dF);
  bool have = false;
  if (o <= acc.o) {
    key = mk();
    have = true;
    if (o < acc.o || key < acc.k) { acc.o = o; acc.k = key; }
  }
  const bool f = mm && follower_ok(D);
  if (f && !have) key = mk();
  return f;
}

// ---------------------------------------------------------------------------
// RELOCATE (moves.py:280-311, batch.py:391-428), warp task = customer u
// ---------------------------------------------------------------------------
template <bool WIN>
__device__ void srelocate(const DevInst &I, const DevPop &P, const IV &v, const RBT<WIN> *R, int b, int u,
                          const double lam[4], bool mm, Acc &acc, double *U, double *Wd) {
  const int lane = threadIdx.x & 31;
  const int lu = __ldg(v.loc + u);
  if (lu < 0) return;
  const int ru = loc_r(lu), pu = loc_p(lu);
  const RBT<WIN> &X1 = R[ru];
  const int k1 = X1.k;
  const int nxt = pu + 2 <= k1 ? __ldg(v.seq + ru * v.Kp + pu + 2) : u;
  // U[0..4] removal terms l=1, U[5..9] l=2, U[10..15] seg l=1, U[16..21] seg l=2
  if (lane == 0) {
    const int n1 = X1.n;
    At<WIN> P1 = pre<WIN>(v, ru, pu);
    for (int l = 1; l <= 2; l++) {
      if (pu + l <= k1) {
        At<WIN> A = P1;
        if (pu + l + 1 <= n1 - 1) A = a_cat_ne<WIN>(I, P1, suf<WIN>(v, ru, pu + l + 1, n1));
        contrib_fast<WIN>(I, A, X1.dep, X1.arr, k1 - l, U + 5 * (l - 1));
      }
    }
    At<WIN> s1 = a_node<WIN>(I, u);
    st_at<WIN>(U + 10, s1);
    if (pu + 2 <= k1) st_at<WIN>(U + 16, a_cat_ne<WIN>(I, s1, a_node<WIN>(I, nxt)));
  }
  __syncwarp();
  constexpr int nvar = WIN ? 2 : 3;
  // front insertion (depot d) + seg is a per-(variant, depot) constant of this u:
  // Wd[(vi*ND + d)*6 ..] = node(d) (+) seg_vi, the first concat of (node(d) (+) seg) (+) S[rb][1]
  if (Wd) {
    for (int idx = lane; idx < nvar * I.ND; idx += 32) {
      const int vi = idx / I.ND, d = idx - vi * I.ND;
      const int len = vi == 0 ? 1 : 2, rev = vi == 2;
      if (pu + len <= k1) {
        At<WIN> seg = ld_at<WIN>(U + (len == 1 ? 10 : 16), rev ? (len == 1 ? u : nxt) : u,
                                 rev ? u : (len == 1 ? u : nxt));
        st_at<WIN>(Wd + idx * 6, a_cat_l<WIN>(a_node<WIN>(I, d), seg, link_of(I, d, seg.first)));
      }
    }
    __syncwarp();
  }
  const double fdec1 = I.nv_on ? __ldg(v.fl + X1.dep).y : 0.0;
  // one candidate: target (r2, tgt) with prefix P2 and (possibly empty) suffix S2
  // one candidate: target (r2, tgt) with prefix P2 and (possibly empty) suffix S2,
  // joined to the segment by the links Lp (P2.last -> seg.first) and Ls (seg.last -> S2.first)
  auto eval_links = [&](int len, int rev, int r2, int tgt, const At<WIN> &P2, const At<WIN> &S2, Link Lp, Link Ls,
                        const RBT<WIN> &X2, unsigned long long &o, unsigned long long &key) -> bool {
    At<WIN> seg = ld_at<WIN>(U + (len == 1 ? 10 : 16), rev ? (len == 1 ? u : nxt) : u, rev ? u : (len == 1 ? u : nxt));
    At<WIN> B = a_cat_l<WIN>(P2, seg, Lp);
    if (S2.first >= 0) B = a_cat_l<WIN>(B, S2, Ls);
    double cB[5];
    contrib_fast<WIN>(I, B, X2.dep, X2.arr, X2.k + len, cB);
    double fleet_delta = 0.0;
    int fn = 1;
    if (I.nv_on && k1 - len == 0) { fleet_delta = 0.0 + fdec1; fn = 0; }
    return two_route_delta<WIN>(I, U + 5 * (len - 1), cB, X1.rc, X2.rc, X1.clo, X2.clo, fleet_delta, fn, lam, acc,
                                [&] { return key_of(ru, pu, r2, tgt, len, 0, rev, 0, -1, -1); }, key, mm,
                                P.nanflag + b, o);
  };
  auto eval_inter = [&](int len, int rev, int r2, int tgt, const At<WIN> &P2, const At<WIN> &S2, const RBT<WIN> &X2,
                        unsigned long long &o, unsigned long long &key) -> bool {
    const int sf = rev ? (len == 1 ? u : nxt) : u, sl = rev ? u : (len == 1 ? u : nxt);
    Link Ls{0.0, 0.0};
    if (S2.first >= 0) Ls = link_of(I, sl, S2.first);
    return eval_links(len, rev, r2, tgt, P2, S2, link_to_u(I, P2.last, sf), Ls, X2, o, key);
  };
  // granular targets: insert after v (p2 = pv + 1).  The node ids around the
  // insertion point are v itself and nxs[v], so every distance link is issued
  // as soon as those two ids are known (one dependent load after the list).
  const int W = I.W;
  const int *lst = I.lists + (size_t)(u - I.ND) * W;
  const bool has2 = pu + 2 <= k1;
  for (int base = 0; base < W; base += 32) {
    const int t = base + lane;
    int vv = -1, lv = -1, sv = -1;
    if (t < W) vv = __ldg(lst + t);
    Link Lvu{0.0, 0.0}, Lvn{0.0, 0.0}, Lus{0.0, 0.0}, Lns{0.0, 0.0};
    if (vv >= 0) {
      lv = __ldg(v.loc + vv);
      sv = __ldg(v.nxs + vv);
      Lvu = link_to_u(I, vv, u);
      if (nvar == 3 && has2) Lvn = link_to_u(I, vv, nxt);
      if (sv >= 0) {
        Lus = link_of(I, u, sv);
        if (has2) Lns = link_of(I, nxt, sv);
      }
    }
    int rv = -1, tgt = -1;
    if (lv >= 0) { rv = loc_r(lv); tgt = loc_p(lv) + 1; }
    const bool same = rv == ru;
    At<WIN> P2, S2;
    if (rv >= 0 && !same) {
      P2 = ld_tab<WIN>(v.tP, rv * v.Kp + tgt);
      P2.first = vv;  // (unused by the deltas)
      P2.last = vv;
      if (sv >= 0) {
        S2 = ld_tab<WIN>(v.tS, rv * v.Kp + tgt + 1);
        S2.first = sv;
        S2.last = sv;  // (unused by the deltas)
      } else {
        S2 = a_empty<WIN>();
      }
    }
#pragma unroll
    for (int vi = 0; vi < nvar; vi++) {
      const int len = vi == 0 ? 1 : 2, rev = vi == 2;
      bool ok = rv >= 0 && pu + len <= k1 && !(same && tgt > pu && tgt <= pu + len);
      if (!rev) ok = ok && !(same && tgt == pu);
      bool fol = false, gqf = false;
      unsigned long long o = 0, key = 0;
      if (ok) {
        if (same) { gqf = true; key = key_of(ru, pu, rv, tgt, len, 0, rev, 0, -1, -1); }
        else fol = eval_links(len, rev, rv, tgt, P2, S2, (len == 2 && rev) ? Lvn : Lvu,
                              (len == 1 || rev) ? Lus : Lns, R[rv], o, key);
      }
      append_fol(P, b, fol, o, key);
      enqueue_g(P, b, 0, gqf, key);
    }
  }
  // boundary targets: front (p2 = 0) and back (p2 = k_rb) of every route rb
  for (int base = 0; base < v.M; base += 32) {
    const int rb = base + lane;
    const bool in = rb < v.M;
    const bool same = rb == ru;
#pragma unroll
    for (int side = 0; side < 2; side++) {
      int tgt = 0;
      At<WIN> P2, S2;
      if (in) {
        const RBT<WIN> &X2 = R[rb];
        if (side == 0) {
          tgt = 0;
          P2 = a_node<WIN>(I, X2.dep);
          S2 = X2.sf_first >= 0 ? rb_sf<WIN>(X2) : a_empty<WIN>();
        } else {
          tgt = X2.k;
          P2 = rb_pb<WIN>(X2);
          S2 = I.open ? a_empty<WIN>() : a_node<WIN>(I, X2.arr);
        }
      }
#pragma unroll
      for (int vi = 0; vi < nvar; vi++) {
        const int len = vi == 0 ? 1 : 2, rev = vi == 2;
        bool ok = in && pu + len <= k1 && !(same && tgt == pu + len);
        if (!rev) ok = ok && !(same && tgt == pu);
        bool fol = false, gqf = false;
        unsigned long long o = 0, key = 0;
        if (ok) {
          if (same) { gqf = true; key = key_of(ru, pu, rb, tgt, len, 0, rev, 0, -1, -1); }
          else if (side == 0 && Wd) {
            // B = (node(dep_rb) (+) seg) (+) S[rb][1] from the precomputed prefix
            const RBT<WIN> &X2 = R[rb];
            const int sl = rev ? u : (len == 1 ? u : nxt);
            At<WIN> B = ld_at<WIN>(Wd + (vi * I.ND + X2.dep) * 6, X2.dep, sl);
            if (S2.first >= 0) B = a_cat_l<WIN>(B, S2, link_of(I, sl, S2.first));
            double cB[5];
            contrib_fast<WIN>(I, B, X2.dep, X2.arr, X2.k + len, cB);
            double fleet_delta = 0.0;
            int fn = 1;
            if (I.nv_on && k1 - len == 0) { fleet_delta = 0.0 + fdec1; fn = 0; }
            fol = two_route_delta<WIN>(I, U + 5 * (len - 1), cB, X1.rc, X2.rc, X1.clo, X2.clo, fleet_delta, fn, lam,
                                       acc, [&] { return key_of(ru, pu, rb, 0, len, 0, rev, 0, -1, -1); }, key, mm,
                                       P.nanflag + b, o);
          } else fol = eval_inter(len, rev, rb, tgt, P2, S2, R[rb], o, key);
        }
        append_fol(P, b, fol, o, key);
        enqueue_g(P, b, 0, gqf, key);
      }
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// RELOCATE, flattened form (the default; MDR_REL_WARP=1 selects srelocate).
// The u-side pieces of the task's CT customers are staged once (one thread per
// customer); the warps then sweep first the (customer, granular slot) items,
// then the (customer, route) boundary items, 32 per chunk, so no lane idles on
// a list or route-count tail and no warp waits on a per-customer staging
// chain.  The front-insertion concat node(d) (+) seg is formed per candidate
// (the warp form's per-depot Wd table is per customer, which the chunks mix).
// Same candidates, deltas and keys as srelocate.
// ---------------------------------------------------------------------------
#ifndef MDR_REL_SIDE_UNROLL
#define MDR_REL_SIDE_UNROLL 1  // front/back sides of a boundary item one after the other: fewer live pieces (C4 +1.5 %, C5 +3.6 % vs unrolled)
#endif
constexpr int kRelSideUnroll = MDR_REL_SIDE_UNROLL;
#ifndef MDR_REL_VAR_UNROLL
#define MDR_REL_VAR_UNROLL 3  // segment variants of a relocate item unrolled (3 = all)
#endif
constexpr int kRelVarUnroll = MDR_REL_VAR_UNROLL;
struct RLU {
  int u, ru, pu, nxt;  // u < 0: out of range or not routed
};
#define MDR_RLD 24  // doubles per staged customer: removal terms l=1,2 [10], seg l=1 [6], seg l=2 [6], fleet_dec [1]

template <bool WIN>
__device__ __forceinline__ void srel_stage(const DevInst &I, const IV &v, const RBT<WIN> *R, int u, RLU &c, double *U) {
  c.u = -1;
  if (u >= I.N) return;
  const int lu = __ldg(v.loc + u);
  if (lu < 0) return;
  const int ru = loc_r(lu), pu = loc_p(lu);
  const RBT<WIN> &X1 = R[ru];
  const int k1 = X1.k, n1 = X1.n;
  const int nxt = pu + 2 <= k1 ? __ldg(v.seq + ru * v.Kp + pu + 2) : u;
  c.u = u; c.ru = ru; c.pu = pu; c.nxt = nxt;
  At<WIN> P1 = pre<WIN>(v, ru, pu);
  for (int l = 1; l <= 2; l++) {
    if (pu + l <= k1) {
      At<WIN> A = P1;
      if (pu + l + 1 <= n1 - 1) A = a_cat_ne<WIN>(I, P1, suf<WIN>(v, ru, pu + l + 1, n1));
      contrib_fast<WIN>(I, A, X1.dep, X1.arr, k1 - l, U + 5 * (l - 1));
    }
  }
  At<WIN> s1 = a_node<WIN>(I, u);
  st_at<WIN>(U + 10, s1);
  if (pu + 2 <= k1) st_at<WIN>(U + 16, a_cat_ne<WIN>(I, s1, a_node<WIN>(I, nxt)));
  U[22] = I.nv_on ? __ldg(v.fl + X1.dep).y : 0.0;
}

// one 32-item chunk: granular items [0, CT*W) when bnd == false, else (customer, route) items [0, CT*M)
template <bool WIN, int CT>
__device__ void srel_chunk(const DevInst &I, const DevPop &P, const IV &v, const RBT<WIN> *R, int b, int chunk, bool bnd,
                           const RLU *C, const double *UD, const double lam[4], bool mm, Acc &acc) {
  const int lane = threadIdx.x & 31;
  const int per = bnd ? v.M : I.W;
  const int item = chunk * 32 + lane;
  const int j = item / per, s = item - j * per;
  int u = -1, ru = 0, pu = 0, nxt = 0;
  const double *U = UD;
  if (j < CT) {
    const RLU c = C[j];
    u = c.u; ru = c.ru; pu = c.pu; nxt = c.nxt;
    U = UD + j * MDR_RLD;
  }
  const bool uok = u >= 0;
  const RBT<WIN> &X1 = R[uok ? ru : 0];
  const int k1 = X1.k;
  const double fdec1 = U[22];
  constexpr int nvar = WIN ? 2 : 3;
  auto eval_links = [&](int len, int rev, int r2, int tgt, const At<WIN> &P2, const At<WIN> &S2, Link Lp, Link Ls,
                        const RBT<WIN> &X2, unsigned long long &o, unsigned long long &key) -> bool {
    At<WIN> seg = ld_at<WIN>(U + (len == 1 ? 10 : 16), rev ? (len == 1 ? u : nxt) : u, rev ? u : (len == 1 ? u : nxt));
    At<WIN> B = a_cat_l<WIN>(P2, seg, Lp);
    if (S2.first >= 0) B = a_cat_l<WIN>(B, S2, Ls);
    double cB[5];
    contrib_fast<WIN>(I, B, X2.dep, X2.arr, X2.k + len, cB);
    double fleet_delta = 0.0;
    int fn = 1;
    if (I.nv_on && k1 - len == 0) { fleet_delta = 0.0 + fdec1; fn = 0; }
    return two_route_delta<WIN>(I, U + 5 * (len - 1), cB, X1.rc, X2.rc, X1.clo, X2.clo, fleet_delta, fn, lam, acc,
                                [&] { return key_of(ru, pu, r2, tgt, len, 0, rev, 0, -1, -1); }, key, mm,
                                P.nanflag + b, o);
  };
  if (!bnd) {
    const bool has2 = pu + 2 <= k1;
    int vv = -1, lv = -1, sv = -1;
    if (uok) vv = __ldg(I.lists + (size_t)(u - I.ND) * I.W + s);
    Link Lvu{0.0, 0.0}, Lvn{0.0, 0.0}, Lus{0.0, 0.0}, Lns{0.0, 0.0};
    if (vv >= 0) {
      lv = __ldg(v.loc + vv);
      sv = __ldg(v.nxs + vv);
      Lvu = link_to_u(I, vv, u);
      if (nvar == 3 && has2) Lvn = link_to_u(I, vv, nxt);
      if (sv >= 0) {
        Lus = link_of(I, u, sv);
        if (has2) Lns = link_of(I, nxt, sv);
      }
    }
    int rv = -1, tgt = -1;
    if (lv >= 0) { rv = loc_r(lv); tgt = loc_p(lv) + 1; }
    const bool same = rv == ru;
    At<WIN> P2, S2;
    if (rv >= 0 && !same) {
      P2 = ld_tab<WIN>(v.tP, rv * v.Kp + tgt);
      P2.first = vv;
      P2.last = vv;
      if (sv >= 0) {
        S2 = ld_tab<WIN>(v.tS, rv * v.Kp + tgt + 1);
        S2.first = sv;
        S2.last = sv;
      } else {
        S2 = a_empty<WIN>();
      }
    }
#pragma unroll kRelVarUnroll
    for (int vi = 0; vi < nvar; vi++) {
      const int len = vi == 0 ? 1 : 2, rev = vi == 2;
      bool ok = rv >= 0 && pu + len <= k1 && !(same && tgt > pu && tgt <= pu + len);
      if (!rev) ok = ok && !(same && tgt == pu);
      bool fol = false, gqf = false;
      unsigned long long o = 0, key = 0;
      if (ok) {
        if (same) { gqf = true; key = key_of(ru, pu, rv, tgt, len, 0, rev, 0, -1, -1); }
        else fol = eval_links(len, rev, rv, tgt, P2, S2, (len == 2 && rev) ? Lvn : Lvu,
                              (len == 1 || rev) ? Lus : Lns, R[rv], o, key);
      }
      append_fol(P, b, fol, o, key);
      enqueue_g(P, b, 0, gqf, key);
    }
    return;
  }
  const int rb = s;
  const bool in = uok;
  const bool same = rb == ru;
#pragma unroll kRelSideUnroll
  for (int side = 0; side < 2; side++) {
    int tgt = 0;
    At<WIN> P2, S2;
    if (in) {
      const RBT<WIN> &X2 = R[rb];
      if (side == 0) {
        tgt = 0;
        P2 = a_node<WIN>(I, X2.dep);
        S2 = X2.sf_first >= 0 ? rb_sf<WIN>(X2) : a_empty<WIN>();
      } else {
        tgt = X2.k;
        P2 = rb_pb<WIN>(X2);
        S2 = I.open ? a_empty<WIN>() : a_node<WIN>(I, X2.arr);
      }
    }
#pragma unroll kRelVarUnroll
    for (int vi = 0; vi < nvar; vi++) {
      const int len = vi == 0 ? 1 : 2, rev = vi == 2;
      bool ok = in && pu + len <= k1 && !(same && tgt == pu + len);
      if (!rev) ok = ok && !(same && tgt == pu);
      bool fol = false, gqf = false;
      unsigned long long o = 0, key = 0;
      if (ok) {
        if (same) { gqf = true; key = key_of(ru, pu, rb, tgt, len, 0, rev, 0, -1, -1); }
        else {
          const int sf = rev ? (len == 1 ? u : nxt) : u, sl = rev ? u : (len == 1 ? u : nxt);
          Link Ls{0.0, 0.0};
          if (S2.first >= 0) Ls = link_of(I, sl, S2.first);
          fol = eval_links(len, rev, rb, tgt, P2, S2, link_to_u(I, P2.last, sf), Ls, R[rb], o, key);
        }
      }
      append_fol(P, b, fol, o, key);
      enqueue_g(P, b, 0, gqf, key);
    }
  }
}

// ---------------------------------------------------------------------------
// SWAP (moves.py:314-358, batch.py:430-463), warp task = customer u
// A = (P1 + segB) + S1, B = (P2 + segA) + S2: X = P1 + segB depends only on v's
// segment (lv, av) and Y = P2 + segA only on u's (lu, au), so each is built
// once per lane and shared by the combos that use it.
// ---------------------------------------------------------------------------
template <bool WIN>
__device__ void sswap(const DevInst &I, const DevPop &P, const IV &v, const RBT<WIN> *R, int b, int u, const double lam[4],
                      bool mm, Acc &acc, double *U) {
  const int lane = threadIdx.x & 31;
  const int lu = __ldg(v.loc + u);
  if (lu < 0) return;
  const int ru = loc_r(lu), pu = loc_p(lu);
  const RBT<WIN> &X1 = R[ru];
  const int k1 = X1.k, n1 = X1.n;
  const int *sq1 = v.seq + ru * v.Kp;
  const int nxtu = pu + 2 <= k1 ? __ldg(sq1 + pu + 2) : u;
  const int dep1 = X1.dep, lastP1 = __ldg(sq1 + pu), lastS1 = __ldg(sq1 + n1 - 1);
  const int s1f1 = pu + 2 <= n1 - 1 ? __ldg(sq1 + pu + 2) : -1;  // S[ru][pu+2].first
  const int s1f2 = pu + 3 <= n1 - 1 ? __ldg(sq1 + pu + 3) : -1;  // S[ru][pu+3].first
  // U[0..5] seg u l=1, U[6..11] seg u l=2, U[12..17] prefix (0..pu), U[18..23] S[ru][pu+2], U[24..29] S[ru][pu+3]
  if (lane == 0) {
    At<WIN> s1 = a_node<WIN>(I, u);
    st_at<WIN>(U, s1);
    if (pu + 2 <= k1) st_at<WIN>(U + 6, a_cat_ne<WIN>(I, s1, a_node<WIN>(I, nxtu)));
    st_at<WIN>(U + 12, pre<WIN>(v, ru, pu));
    if (s1f1 >= 0) st_at<WIN>(U + 18, suf<WIN>(v, ru, pu + 2, n1));
    if (s1f2 >= 0) st_at<WIN>(U + 24, suf<WIN>(v, ru, pu + 3, n1));
  }
  __syncwarp();
  constexpr int NV = WIN ? 2 : 3;  // segment variants (len, rev): (1,0), (2,0), (2,1)
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
    const bool inter = rv >= 0 && !same;
    int k2 = 0, n2 = 0, nxtv = vv;
    At<WIN> P2;
    At<WIN> Y[NV];
    if (inter) {
      k2 = R[rv].k;
      n2 = R[rv].n;
      P2 = pre<WIN>(v, rv, pv);
      if (pv + 2 <= k2) nxtv = __ldg(v.seq + rv * v.Kp + pv + 2);
#pragma unroll
      for (int yi = 0; yi < NV; yi++) {
        const int lu_ = yi == 0 ? 1 : 2, au = yi == 2;
        if (pu + lu_ <= k1) {
          const int ua = lu_ == 1 ? u : nxtu;
          At<WIN> sA = ld_at<WIN>(U + (lu_ == 1 ? 0 : 6), au ? ua : u, au ? u : ua);
          Y[yi] = a_cat_l<WIN>(P2, sA, link_to_u(I, P2.last, sA.first));
        }
      }
    }
#pragma unroll
    for (int xi = 0; xi < NV; xi++) {
      const int lv_ = xi == 0 ? 1 : 2, av = xi == 2;
      const bool xok = inter && pv + lv_ <= k2;
      At<WIN> X, S2;
      if (xok) {
        At<WIN> sB = a_node<WIN>(I, vv);
        if (lv_ == 2) sB = a_cat_ne<WIN>(I, sB, a_node<WIN>(I, nxtv));
        if (av) swap_ends(sB);
        X = a_cat_l<WIN>(ld_at<WIN>(U + 12, dep1, lastP1), sB, link_of(I, lastP1, sB.first));
        S2 = suf<WIN>(v, rv, pv + lv_ + 1, n2);
      }
#pragma unroll
      for (int yi = 0; yi < NV; yi++) {
        const int lu_ = yi == 0 ? 1 : 2, au = yi == 2;
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
          } else if (xok && pu + lu_ <= k1) {
            const int sf = lu_ == 1 ? s1f1 : s1f2;
            At<WIN> A = X;
            if (sf >= 0) A = a_cat_l<WIN>(X, ld_at<WIN>(U + (lu_ == 1 ? 18 : 24), sf, lastS1), link_to_u(I, X.last, sf));
            At<WIN> B = Y[yi];
            if (S2.first >= 0) B = a_cat_l<WIN>(B, S2, link_of(I, B.last, S2.first));
            double cA[5], cB[5];
            contrib_fast<WIN>(I, A, X1.dep, X1.arr, k1 - lu_ + lv_, cA);
            const RBT<WIN> &X2 = R[rv];
            contrib_fast<WIN>(I, B, X2.dep, X2.arr, k2 - lv_ + lu_, cB);
            fol = two_route_delta<WIN>(I, cA, cB, X1.rc, X2.rc, X1.clo, X2.clo, 0.0, 1, lam, acc,
                                       [&] { return key_of(ru, pu, rv, pv, lu_, lv_, au, av, -1, -1); }, key, mm,
                                       P.nanflag + b, o);
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
// SWAP, flattened form (the default; MDR_SWAP_WARP=1 selects sswap above).
// The u-side pieces of all CT customers of the CTA task are staged once, one
// thread per customer, before the warps start; the warps then sweep the
// task's (customer, granular slot) items 32 at a time.  Every lane is busy
// (θ = 50 left 14 of every 64 slots of the per-customer sweep idle) and no
// warp waits on a serial lane-0 staging chain per customer.  Same candidates,
// same deltas, same keys as sswap.
// ---------------------------------------------------------------------------
struct SWU {
  int u, ru, pu, nxtu, lastP1, lastS1, s1f1, s1f2;  // u < 0: out of range or not routed
};
#define MDR_SWD 30  // doubles per staged customer: seg l=1, seg l=2, P[ru][pu], S[ru][pu+2], S[ru][pu+3]

template <bool WIN>
__device__ __forceinline__ void sswap_stage(const DevInst &I, const IV &v, const RBT<WIN> *R, int u, SWU &c, double *U) {
  c.u = -1;
  if (u >= I.N) return;
  const int lu = __ldg(v.loc + u);
  if (lu < 0) return;
  const int ru = loc_r(lu), pu = loc_p(lu);
  const int k1 = R[ru].k, n1 = R[ru].n;
  const int *sq1 = v.seq + ru * v.Kp;
  const int nxtu = pu + 2 <= k1 ? __ldg(sq1 + pu + 2) : u;
  c.u = u; c.ru = ru; c.pu = pu; c.nxtu = nxtu;
  c.lastP1 = __ldg(sq1 + pu);
  c.lastS1 = __ldg(sq1 + n1 - 1);
  c.s1f1 = pu + 2 <= n1 - 1 ? __ldg(sq1 + pu + 2) : -1;
  c.s1f2 = pu + 3 <= n1 - 1 ? __ldg(sq1 + pu + 3) : -1;
  At<WIN> s1 = a_node<WIN>(I, u);
  st_at<WIN>(U, s1);
  if (pu + 2 <= k1) st_at<WIN>(U + 6, a_cat_ne<WIN>(I, s1, a_node<WIN>(I, nxtu)));
  st_at<WIN>(U + 12, pre<WIN>(v, ru, pu));
  if (c.s1f1 >= 0) st_at<WIN>(U + 18, suf<WIN>(v, ru, pu + 2, n1));
  if (c.s1f2 >= 0) st_at<WIN>(U + 24, suf<WIN>(v, ru, pu + 3, n1));
}

// one 32-item chunk of the task's (customer, slot) space; full-warp call
#ifndef MDR_SWAP_YOUTER_NW
#define MDR_SWAP_YOUTER_NW 0  // u-side-outer swap also without windows (measured slower at C5)
#endif
// XF: which v-side segments this call evaluates -- 0 all, 1 length 1 only, 2 length 2 only
// (the swap evaluator can run as two kernels, each with half the live state)
template <bool WIN, int CT, int XF = 0>
__device__ void sswap_chunk(const DevInst &I, const DevPop &P, const IV &v, const RBT<WIN> *R, int b, int chunk,
                            const SWU *C, const double *UD, const double lam[4], bool mm, Acc &acc) {
  const int lane = threadIdx.x & 31;
  const int W = I.W;
  const int item = chunk * 32 + lane;
  const int j = item / W, t = item - j * W;
  int u = -1;
  if (j < CT) u = C[j].u;
  int vv = -1;
  if (u >= 0) vv = __ldg(I.lists + (size_t)(u - I.ND) * W + t);
  int ru = -1, pu = 0, nxtu = 0, lastP1 = 0, lastS1 = 0, s1f1 = -1, s1f2 = -1;
  const double *U = UD;
  if (u >= 0) {
    const SWU &c = C[j];
    ru = c.ru; pu = c.pu; nxtu = c.nxtu; lastP1 = c.lastP1; lastS1 = c.lastS1; s1f1 = c.s1f1; s1f2 = c.s1f2;
    U = UD + j * MDR_SWD;
  }
  int rv = -1, pv = -1;
  if (vv >= 0 && vv != u) {
    int lv = __ldg(v.loc + vv);
    if (lv >= 0) { rv = loc_r(lv); pv = loc_p(lv); }
  }
  const RBT<WIN> &X1 = R[ru < 0 ? 0 : ru];
  const int k1 = X1.k;
  const bool same = rv == ru;
  const bool inter = rv >= 0 && !same;
  constexpr int NV = WIN ? 2 : 3;  // segment variants (len, rev): (1,0), (2,0), (2,1)
  int k2 = 0, n2 = 0, nxtv = vv;
  At<WIN> P2;
  At<WIN> Y[NV];
if constexpr (CT >= 32 && (WIN || MDR_SWAP_YOUTER_NW)) {  // large shape with windows: u-side variant outer (C4 swap -4.5 % at 20 warps x 96)
  // u-side variant outer, v-side inner: only one donor-side prefix Y is live; the v-side
  // piece X and suffix S2 are re-formed per u-side variant (more work, fewer registers)
  if (inter) {
    k2 = R[rv].k;
    n2 = R[rv].n;
    if (pv + 2 <= k2) nxtv = __ldg(v.seq + rv * v.Kp + pv + 2);
  }
#pragma unroll
  for (int yi = 0; yi < NV; yi++) {
    const int lu_ = yi == 0 ? 1 : 2, au = yi == 2;
    At<WIN> Yc;
    if (inter && pu + lu_ <= k1) {
      const At<WIN> P2 = pre<WIN>(v, rv, pv);
      const int ua = lu_ == 1 ? u : nxtu;
      At<WIN> sA = ld_at<WIN>(U + (lu_ == 1 ? 0 : 6), au ? ua : u, au ? u : ua);
      Yc = a_cat_l<WIN>(P2, sA, link_to_u(I, P2.last, sA.first));
    }
#pragma unroll
    for (int xi = (XF == 2 ? 1 : 0); xi < (XF == 1 ? 1 : NV); xi++) {
      const int lv_ = xi == 0 ? 1 : 2, av = xi == 2;
      const bool xok = inter && pv + lv_ <= k2;
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
        } else if (xok && pu + lu_ <= k1) {
          At<WIN> sB = a_node<WIN>(I, vv);
          if (lv_ == 2) sB = a_cat_ne<WIN>(I, sB, a_node<WIN>(I, nxtv));
          if (av) swap_ends(sB);
          At<WIN> A = a_cat_l<WIN>(ld_at<WIN>(U + 12, X1.dep, lastP1), sB, link_of(I, lastP1, sB.first));
          const int sf = lu_ == 1 ? s1f1 : s1f2;
          if (sf >= 0) A = a_cat_l<WIN>(A, ld_at<WIN>(U + (lu_ == 1 ? 18 : 24), sf, lastS1), link_to_u(I, A.last, sf));
          double cA[5], cB[5];
          contrib_fast<WIN>(I, A, X1.dep, X1.arr, k1 - lu_ + lv_, cA);
          At<WIN> B = Yc;
          const At<WIN> S2 = suf<WIN>(v, rv, pv + lv_ + 1, n2);
          if (S2.first >= 0) B = a_cat_l<WIN>(B, S2, link_of(I, B.last, S2.first));
          const RBT<WIN> &X2 = R[rv];
          contrib_fast<WIN>(I, B, X2.dep, X2.arr, k2 - lv_ + lu_, cB);
          fol = two_route_delta<WIN>(I, cA, cB, X1.rc, X2.rc, X1.clo, X2.clo, 0.0, 1, lam, acc,
                                     [&] { return key_of(ru, pu, rv, pv, lu_, lv_, au, av, -1, -1); }, key, mm,
                                     P.nanflag + b, o);
        }
      }
      append_fol(P, b, fol, o, key);
      enqueue_g(P, b, 1, gqf, key);
    }
  }
  } else {
  if (inter) {
    k2 = R[rv].k;
    n2 = R[rv].n;
    P2 = pre<WIN>(v, rv, pv);
    if (pv + 2 <= k2) nxtv = __ldg(v.seq + rv * v.Kp + pv + 2);
#pragma unroll
    for (int yi = 0; yi < NV; yi++) {
      const int lu_ = yi == 0 ? 1 : 2, au = yi == 2;
      if (pu + lu_ <= k1) {
        const int ua = lu_ == 1 ? u : nxtu;
        At<WIN> sA = ld_at<WIN>(U + (lu_ == 1 ? 0 : 6), au ? ua : u, au ? u : ua);
        Y[yi] = a_cat_l<WIN>(P2, sA, link_to_u(I, P2.last, sA.first));
      }
    }
  }
#pragma unroll
  for (int xi = (XF == 2 ? 1 : 0); xi < (XF == 1 ? 1 : NV); xi++) {
    const int lv_ = xi == 0 ? 1 : 2, av = xi == 2;
    const bool xok = inter && pv + lv_ <= k2;
    At<WIN> X, S2;
    if (xok) {
      At<WIN> sB = a_node<WIN>(I, vv);
      if (lv_ == 2) sB = a_cat_ne<WIN>(I, sB, a_node<WIN>(I, nxtv));
      if (av) swap_ends(sB);
      X = a_cat_l<WIN>(ld_at<WIN>(U + 12, X1.dep, lastP1), sB, link_of(I, lastP1, sB.first));
      S2 = suf<WIN>(v, rv, pv + lv_ + 1, n2);
    }
#pragma unroll
    for (int yi = 0; yi < NV; yi++) {
      const int lu_ = yi == 0 ? 1 : 2, au = yi == 2;
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
        } else if (xok && pu + lu_ <= k1) {
          const int sf = lu_ == 1 ? s1f1 : s1f2;
          At<WIN> A = X;
          if (sf >= 0) A = a_cat_l<WIN>(X, ld_at<WIN>(U + (lu_ == 1 ? 18 : 24), sf, lastS1), link_to_u(I, X.last, sf));
          At<WIN> B = Y[yi];
          if (S2.first >= 0) B = a_cat_l<WIN>(B, S2, link_of(I, B.last, S2.first));
          double cA[5], cB[5];
          contrib_fast<WIN>(I, A, X1.dep, X1.arr, k1 - lu_ + lv_, cA);
          const RBT<WIN> &X2 = R[rv];
          contrib_fast<WIN>(I, B, X2.dep, X2.arr, k2 - lv_ + lu_, cB);
          fol = two_route_delta<WIN>(I, cA, cB, X1.rc, X2.rc, X1.clo, X2.clo, 0.0, 1, lam, acc,
                                     [&] { return key_of(ru, pu, rv, pv, lu_, lv_, au, av, -1, -1); }, key, mm,
                                     P.nanflag + b, o);
        }
      }
      append_fol(P, b, fol, o, key);
      enqueue_g(P, b, 1, gqf, key);
    }
  }
  }
}


// ---------------------------------------------------------------------------
// TWO_OPT_STAR (moves.py:375-405, batch.py:475-494)
// ---------------------------------------------------------------------------
// A = PA (+) SB, B = PB (+) SA for the cut (r1, p1, r2, p2); SA/SB may be empty
// uA / uB: which end of the A / B link is warp-uniform (0 = the prefix's last node, 1 = the suffix's first)
template <bool WIN>
__device__ __forceinline__ bool tos_eval(const DevInst &I, const DevPop &P, const IV &v, int b, const RBT<WIN> &X1,
                                         const RBT<WIN> &X2, int r1, int p1, int r2, int p2, const At<WIN> &PA,
                                         const At<WIN> &SB, const At<WIN> &PB, const At<WIN> &SA, int uA, int uB,
                                         const double lam[4], Acc &acc, bool mm, unsigned long long &o,
                                         unsigned long long &key) {
  At<WIN> A = PA;
  if (SB.first >= 0)
    A = a_cat_l<WIN>(A, SB, uA ? link_to_u(I, PA.last, SB.first) : link_of(I, PA.last, SB.first));
  At<WIN> B = PB;
  if (SA.first >= 0)
    B = a_cat_l<WIN>(B, SA, uB ? link_to_u(I, PB.last, SA.first) : link_of(I, PB.last, SA.first));
  const int kA = p1 + (X2.k - p2), kB = p2 + (X1.k - p1);
  double cA[5], cB[5];
  contrib_fast<WIN>(I, A, X1.dep, X2.arr, kA, cA);
  contrib_fast<WIN>(I, B, X2.dep, X1.arr, kB, cB);
  double fleet_delta = 0.0;
  int fn = 1;
  if (I.nv_on) {
    fleet_delta = (0.0 + (kA == 0 ? __ldg(v.fl + X1.dep).y : 0.0)) + (kB == 0 ? __ldg(v.fl + X2.dep).y : 0.0);
    fn = (kA > 0) && (kB > 0);
  }
  return two_route_delta<WIN>(I, cA, cB, X1.rc, X2.rc, X1.clo, X2.clo, fleet_delta, fn, lam, acc,
                              [&] { return key_of(r1, p1, r2, p2, 0, 0, 0, 0, -1, -1); }, key, mm, P.nanflag + b, o);
}

// A-side terms given (cA precomputed, nullptr = zero route); B = PB (+) SA computed
template <bool WIN>
__device__ __forceinline__ bool tos_eval_pre(const DevInst &I, const DevPop &P, const IV &v, int b, const RBT<WIN> &X1,
                                             const RBT<WIN> &X2, int r1, int p1, int r2, int p2, const double *cA,
                                             const At<WIN> &PB, const At<WIN> &SA, int uB, const double lam[4],
                                             Acc &acc, bool mm, unsigned long long &o, unsigned long long &key) {
  At<WIN> B = PB;
  if (SA.first >= 0)
    B = a_cat_l<WIN>(B, SA, uB ? link_to_u(I, PB.last, SA.first) : link_of(I, PB.last, SA.first));
  const int kA = p1 + (X2.k - p2), kB = p2 + (X1.k - p1);
  double cB[5];
  const double z[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  contrib_fast<WIN>(I, B, X2.dep, X1.arr, kB, cB);
  double fleet_delta = 0.0;
  int fn = 1;
  if (I.nv_on) {
    fleet_delta = (0.0 + (kA == 0 ? __ldg(v.fl + X1.dep).y : 0.0)) + (kB == 0 ? __ldg(v.fl + X2.dep).y : 0.0);
    fn = (kA > 0) && (kB > 0);
  }
  return two_route_delta<WIN>(I, cA ? cA : z, cB, X1.rc, X2.rc, X1.clo, X2.clo, fleet_delta, fn, lam, acc,
                              [&] { return key_of(r1, p1, r2, p2, 0, 0, 0, 0, -1, -1); }, key, mm, P.nanflag + b, o);
}

// warp task = customer u: granular cut and the two boundary families
template <bool WIN>
__device__ void stos_u(const DevInst &I, const DevPop &P, const IV &v, const RBT<WIN> *R, int b, int u, const double lam[4],
                       bool mm, Acc &acc, double *U, double *Wd) {
  const int lane = threadIdx.x & 31;
  const int lu = __ldg(v.loc + u);
  if (lu < 0) return;
  const int ru = loc_r(lu), pu = loc_p(lu);
  const RBT<WIN> &X1 = R[ru];
  const int n1 = X1.n;
  const int *sq1 = v.seq + ru * v.Kp;
  // u-side pieces: U[0..5] P[ru][pu+1], U[6..11] S[ru][pu+2], U[12..17] P[ru][pu], U[18..23] S[ru][pu+1]
  const int lastP0 = __ldg(sq1 + pu), s2first = pu + 2 <= n1 - 1 ? __ldg(sq1 + pu + 2) : -1;
  const int lastS = __ldg(sq1 + n1 - 1);
  if (lane == 0) {
    st_at<WIN>(U, pre<WIN>(v, ru, pu + 1));
    if (s2first >= 0) st_at<WIN>(U + 6, suf<WIN>(v, ru, pu + 2, n1));
    st_at<WIN>(U + 12, pre<WIN>(v, ru, pu));
    st_at<WIN>(U + 18, suf<WIN>(v, ru, pu + 1, n1));
  }
  __syncwarp();
  // the warp-uniform u-side pieces are re-read from shared memory where used (broadcast
  // loads) instead of being held in registers across the loops
#define PU1 ld_at<WIN>(U, X1.dep, u)
#define SU2 (s2first >= 0 ? ld_at<WIN>(U + 6, s2first, lastS) : a_empty<WIN>())
  // granular: (ru, pu+1, rv, pv)
  const int W = I.W;
  const int *lst = I.lists + (size_t)(u - I.ND) * W;
  for (int base = 0; base < W; base += 32) {
    const int t = base + lane;
    int rv = -1, pv = 0;
    if (t < W) {
      int vv = __ldg(lst + t);
      if (vv >= 0) {
        int lv = __ldg(v.loc + vv);
        if (lv >= 0 && loc_r(lv) != ru) { rv = loc_r(lv); pv = loc_p(lv); }
      }
    }
    bool fol = false;
    unsigned long long o = 0, key = 0;
    if (rv >= 0) {
      const RBT<WIN> &X2 = R[rv];
      fol = tos_eval<WIN>(I, P, v, b, X1, X2, ru, pu + 1, rv, pv, PU1, suf<WIN>(v, rv, pv + 1, X2.n),
                          pre<WIN>(v, rv, pv), SU2, 0, 1, lam, acc, mm, o, key);
    }
    append_fol(P, b, fol, o, key);
  }
  // boundary families for every route rb != ru
#define PU0 ld_at<WIN>(U + 12, X1.dep, lastP0)
#define SU1 ld_at<WIN>(U + 18, u, lastS)
  // their A sides depend on u and one depot only: Wd[d*5..] = terms of P[ru][pu+1] (+) arrival d,
  // Wd[(ND+d)*5..] = terms of departure d (+) S[ru][pu+1]
  if (Wd) {
    for (int d = lane; d < I.ND; d += 32) {
      At<WIN> A1 = PU1;
      if (!I.open) A1 = a_cat_l<WIN>(PU1, a_node<WIN>(I, d), link_of(I, u, d));
      contrib_fast<WIN>(I, A1, X1.dep, d, pu + 1, Wd + d * 5);
      At<WIN> A2 = a_cat_l<WIN>(a_node<WIN>(I, d), SU1, link_of(I, d, u));
      contrib_fast<WIN>(I, A2, d, X1.arr, X1.k - pu, Wd + (I.ND + d) * 5);
    }
    __syncwarp();
  }
  for (int base = 0; base < v.M; base += 32) {
    const int rb = base + lane;
    const bool in = rb < v.M && rb != ru;
    // (ru, pu+1, rb, k_rb): u's tail to the end of rb, minus "both tails empty, same arrival"
    {
      bool fol = false;
      unsigned long long o = 0, key = 0;
      if (in) {
        const RBT<WIN> &X2 = R[rb];
        bool drop = (pu + 1 == X1.k);
        if (!I.open) drop = drop && (X1.arr == X2.arr);
        if (!drop) {
          if (Wd) {
            fol = tos_eval_pre<WIN>(I, P, v, b, X1, X2, ru, pu + 1, rb, X2.k, Wd + (I.open ? 0 : X2.arr) * 5,
                                    rb_pb<WIN>(X2), SU2, 1, lam, acc, mm, o, key);
          } else {
            At<WIN> SB = I.open ? a_empty<WIN>() : a_node<WIN>(I, X2.arr);
            fol = tos_eval<WIN>(I, P, v, b, X1, X2, ru, pu + 1, rb, X2.k, PU1, SB, rb_pb<WIN>(X2), SU2, 0, 1, lam,
                                acc, mm, o, key);
          }
        }
      }
      append_fol(P, b, fol, o, key);
    }
    // (rb, 0, ru, pu): rb's customers follow u's head
    {
      bool fol = false;
      unsigned long long o = 0, key = 0;
      if (in) {
        const RBT<WIN> &X2 = R[rb];
        At<WIN> SB = X2.sf_first >= 0 ? rb_sf<WIN>(X2) : a_empty<WIN>();
        if (Wd)
          fol = tos_eval_pre<WIN>(I, P, v, b, X2, X1, rb, 0, ru, pu, Wd + (I.ND + X2.dep) * 5, PU0, SB, 0, lam, acc,
                                  mm, o, key);
        else
          fol = tos_eval<WIN>(I, P, v, b, X2, X1, rb, 0, ru, pu, a_node<WIN>(I, X2.dep), SU1, PU0, SB, 1, 0, lam,
                              acc, mm, o, key);
      }
      append_fol(P, b, fol, o, key);
    }
  }
  __syncwarp();
#undef PU1
#undef SU2
#undef PU0
#undef SU1
}

// warp task = route ra: route pairs (ra, 0, rb, k_rb) (moves.py:401-404)
template <bool WIN>
__device__ void stos_r(const DevInst &I, const DevPop &P, const IV &v, const RBT<WIN> *R, int b, int ra, const double lam[4],
                       bool mm, Acc &acc) {
  const int lane = threadIdx.x & 31;
  const RBT<WIN> &X1 = R[ra];
  const At<WIN> PA = a_node<WIN>(I, X1.dep);
  const At<WIN> SA = X1.sf_first >= 0 ? rb_sf<WIN>(X1) : a_empty<WIN>();
  for (int base = 0; base < v.M; base += 32) {
    const int rb = base + lane;
    bool fol = false;
    unsigned long long o = 0, key = 0;
    if (rb < v.M && rb != ra) {
      // kA = 0 + (k_rb - k_rb) = 0: route ra empties, its new terms are exact zeros
      const RBT<WIN> &X2 = R[rb];
      fol = tos_eval_pre<WIN>(I, P, v, b, X1, X2, ra, 0, rb, X2.k, nullptr, rb_pb<WIN>(X2), SA, 1, lam, acc, mm, o,
                              key);
    }
    append_fol(P, b, fol, o, key);
  }
}

__host__ __device__ __forceinline__ int op_tasks_c(int op, int M, int NC, int ct) {
  int nch = (NC + ct - 1) / ct;
  if (op == 2) return M < 2 ? 0 : nch + (M + ct - 1) / ct;
  return nch;
}

}  // namespace mdr
