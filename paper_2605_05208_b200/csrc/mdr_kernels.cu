// mdr_kernels.cu -- sm_100a kernels of the population-batched local search.
//
//   k_rebuild      one CTA per individual: SolutionIndex + subsequence tables
//                  + route contributions + fleet increments (batch.py:51-158)
//   k_plan         one CTA: per individual the operator of this round
//                  (pre-drawn rng.shuffle stream), its candidate index-space
//                  size, and the chunk offsets of the flattened work list
//   k_eval         persistent grid over all individuals' chunks: implicit
//                  enumeration (moves.py) + fp64 evaluation (batch.py:365-553)
//                  + (dF, key) min-reduction + follower compaction
//   k_select       one CTA per individual: leader, greedy route-disjoint
//                  follower selection, apply, drop empties, rebuild, totals,
//                  penalty adaptation, state machine (localsearch.py:97-140)
#include <cstdio>
#include <cstdlib>

#include "mdr_fused.cuh"
#include "mdr_staged.cuh"
#include "mdr_kernels.cuh"

namespace mdr {

// ---------------------------------------------------------------------------
// block helpers
// ---------------------------------------------------------------------------
struct OK {
  unsigned long long o, k;
};
__device__ __forceinline__ bool ok_less(const OK &a, const OK &b) {
  return a.o < b.o || (a.o == b.o && a.k < b.k);
}
__device__ __forceinline__ OK warp_min(OK v) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    OK w;
    w.o = __shfl_xor_sync(0xffffffffu, v.o, s);
    w.k = __shfl_xor_sync(0xffffffffu, v.k, s);
    if (ok_less(w, v)) v = w;
  }
  return v;
}
// block-wide min; result valid in all threads. sm needs blockDim/32 entries.
__device__ __forceinline__ OK block_min(OK v, OK *sm) {
  v = warp_min(v);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  if (w == 0) {
    OK x = l < nw ? sm[l] : OK{~0ull, ~0ull};
    x = warp_min(x);
    if (l == 0) sm[0] = x;
  }
  __syncthreads();
  OK r = sm[0];
  __syncthreads();
  return r;
}

// numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src), field f
// of rcon.  The recursion (halves rounded down to a multiple of 8, blocks of
// <= 128 summed with 8 accumulators) is run with an explicit stack: device
// recursion would overflow the default per-thread stack for long route lists.
__device__ __forceinline__ double pw_leaf(const double4 *a, int f, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; i++) res += (&a[i].x)[f];
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; j++) r[j] = (&a[j].x)[f];
  int i;
  for (i = 8; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; j++) r[j] += (&a[i + j].x)[f];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; i++) res += (&a[i].x)[f];
  return res;
}

__device__ double pw_sum(const double4 *a, int f, int n) {
  if (n <= 128) return pw_leaf(a, f, n);
  int st_start[32], st_n[32], st_n2[32], st_state[32];
  double st_left[32];
  int sp = 0;
  st_start[0] = 0; st_n[0] = n; st_state[0] = 0;
  double ret = 0.0;
  for (;;) {
    const int S = st_start[sp], Nn = st_n[sp];
    if (st_state[sp] == 0) {
      if (Nn <= 128) {
        ret = pw_leaf(a + S, f, Nn);
        if (sp == 0) return ret;
        --sp;
        continue;
      }
      int n2 = Nn / 2;
      n2 -= n2 % 8;
      st_n2[sp] = n2;
      st_state[sp] = 1;
      ++sp;
      st_start[sp] = S; st_n[sp] = n2; st_state[sp] = 0;
    } else if (st_state[sp] == 1) {
      st_left[sp] = ret;
      st_state[sp] = 2;
      const int n2 = st_n2[sp];
      ++sp;
      st_start[sp] = S + n2; st_n[sp] = Nn - n2; st_state[sp] = 0;
    } else {
      ret = st_left[sp] + ret;
      if (sp == 0) return ret;
      --sp;
    }
  }
}

// per-route part: SolutionIndex entries of its customers (warp per route),
// prefix/suffix tables (the left fold from i of batch.py:99-124) and route
// terms.  The folds run on a group of G lanes per route, each lane folding the
// row pair (i, n-1-i) -- n+1 steps per lane -- so a warp rebuilds 32/G routes
// at once.  list == nullptr: all m.
template <bool WIN>
__device__ __forceinline__ void fold_row(const DevInst &I, const DevPop &P, int b, int r, const int *sq, int i, int n,
                                         int4 mt) {
  At<WIN> acc = a_node<WIN>(I, sq[i]);
  double *trow = P.tabT + (row_base(P, b, r) + i) * P.Kp * P.FE;  // T[r][i][*]
  if (i == 0) tab_store<WIN>(P, P.tabP, b, r, 0, acc);
  tab_store_at<WIN>(trow + i * P.FE, acc);
  for (int j = i + 1; j < n; j++) {
    acc = a_cat_ne<WIN>(I, acc, a_node<WIN>(I, sq[j]));
    if (i == 0) tab_store<WIN>(P, P.tabP, b, r, j, acc);
    tab_store_at<WIN>(trow + j * P.FE, acc);
  }
  tab_store<WIN>(P, P.tabS, b, r, i, acc);
  if (i == 0) {
    double o[5];
    contrib<WIN>(I, acc, mt.y, mt.z, mt.x, o);
    P.rcon[(size_t)b * P.J + r] = make_double4(acc.dist, o[1], o[2], o[3]);  // route_D is the raw table value
    P.rmeta[(size_t)b * P.J + r].w = (int)o[4];
  }
}

#ifdef MDR_SEL_PROF
__device__ unsigned long long g_selprof[16];
#define RBT_(i) do { if (threadIdx.x == 0) { long long t__ = clock64(); atomicAdd(&g_selprof[i], (unsigned long long)(t__ - t_rb)); t_rb = t__; } } while (0)
#else
#define RBT_(i) do { } while (0)
#endif
#ifndef MDR_RB_STAGED
#define MDR_RB_STAGED 1  // 0: a warp per route, a lane per row, node/link reads from global memory
#endif
constexpr int kRbGroup = 8;                 // lanes per route in the staged folds
constexpr size_t kRbStageBytes = 32 * 1024;  // staged positions (>= one route of 502 positions)

// route positions staged in shared memory (structure of arrays): the node
// attributes and the link from the previous position, so the folds' serial
// steps read nothing from global memory
template <bool WIN>
struct RbStage {
  double *load, *T, *E, *L, *c, *t;
  int *v;
  int cap;
  __device__ __forceinline__ RbStage(void *buf, size_t bytes) {
    cap = (int)(bytes / ((WIN ? 6 : 4) * sizeof(double) + sizeof(int)));
    double *d = reinterpret_cast<double *>(buf);
    load = d; T = d + cap; c = d + 2 * cap; t = d + 3 * cap;
    E = WIN ? d + 4 * cap : nullptr;
    L = WIN ? d + 5 * cap : nullptr;
    v = reinterpret_cast<int *>(d + (WIN ? 6 : 4) * cap);
  }
  __device__ __forceinline__ At<WIN> node(int x) const {  // == a_node(I, v[x])
    At<WIN> a;
    a.dist = 0.0; a.load = load[x]; a.T = T[x];
    if (WIN) { a.E = E[x]; a.L = L[x]; } else { a.E = 0.0; a.L = 0.0; }
    a.TW = 0.0;
    a.first = v[x]; a.last = v[x];
    return a;
  }
};

// fold of row i from the staged positions base..base+n-1 (same arithmetic as fold_row)
template <bool WIN>
__device__ __forceinline__ void fold_row_s(const DevInst &I, const DevPop &P, int b, int r, const RbStage<WIN> &St,
                                           int base, int i, int n, int4 mt) {
  At<WIN> acc = St.node(base + i);
  double *trow = P.tabT + (row_base(P, b, r) + i) * P.Kp * P.FE;  // T[r][i][*]
  if (i == 0) tab_store<WIN>(P, P.tabP, b, r, 0, acc);
  tab_store_at<WIN>(trow + i * P.FE, acc);
  for (int j = i + 1; j < n; j++) {
    acc = a_cat_l<WIN>(acc, St.node(base + j), Link{St.c[base + j], St.t[base + j]});
    if (i == 0) tab_store<WIN>(P, P.tabP, b, r, j, acc);
    tab_store_at<WIN>(trow + j * P.FE, acc);
  }
  tab_store<WIN>(P, P.tabS, b, r, i, acc);
  if (i == 0) {
    double o[5];
    contrib<WIN>(I, acc, mt.y, mt.z, mt.x, o);
    P.rcon[(size_t)b * P.J + r] = make_double4(acc.dist, o[1], o[2], o[3]);
    P.rmeta[(size_t)b * P.J + r].w = (int)o[4];
  }
}

// whole CTA.  off: shared int[offcap] (route position offsets), stg: shared
// staging buffer of stg_bytes.  Routes are staged in batches that fit; a group
// of kRbGroup lanes folds each route, a lane taking the row pair (i, n-1-i).
template <bool WIN>
__device__ void rebuild_routes(const DevInst &I, const DevPop &P, int b, const int *list, int cnt, int *off,
                               int offcap, void *stg, size_t stg_bytes) {
  int *LOC = P.loc + (size_t)b * P.N;
  int *NXS = P.nxs + (size_t)b * P.N;
  const int4 *RM = P.rmeta + (size_t)b * P.J;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // few routes (the incremental rebuild): a warp per route, one pass
  if (!MDR_RB_STAGED || cnt <= nw || cnt + 1 > offcap || stg == nullptr) {
    for (int q = wid; q < cnt; q += nw) {
      const int r = list ? list[q] : q;
      const int4 mt = RM[r];
      const int k = mt.x, n = k + (I.open ? 1 : 2);
      const int *sq = P.seq + row_base(P, b, r);
      for (int p = lane; p < k; p += 32) {
        LOC[sq[p + 1]] = (r << 9) | p;
        NXS[sq[p + 1]] = p + 2 <= n - 1 ? sq[p + 2] : -1;
      }
      for (int i = lane; i < n; i += 32) fold_row<WIN>(I, P, b, r, sq, i, n, mt);
    }
    return;
  }
#ifdef MDR_SEL_PROF
  long long t_rb = clock64();
#endif
  // position offsets of the routes: lengths loaded by all threads at once, then
  // one warp scans them in shared memory
  for (int q = threadIdx.x; q < cnt; q += blockDim.x) off[q + 1] = RM[list ? list[q] : q].x + (I.open ? 1 : 2);
  __syncthreads();
  if (threadIdx.x < 32) {
    int carry = 0;
    for (int q0 = 0; q0 < cnt; q0 += 32) {
      const int q = q0 + lane;
      int x = q < cnt ? off[q + 1] : 0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      if (q < cnt) off[q + 1] = carry + x;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) off[0] = 0;
  }
  __syncthreads();
  RBT_(12);
  const RbStage<WIN> St(stg, stg_bytes);
  const int gid = threadIdx.x / kRbGroup, ng = blockDim.x / kRbGroup, sub = threadIdx.x % kRbGroup;
  for (int q0 = 0; q0 < cnt;) {
    int lo = q0 + 1, hi = cnt;  // routes q0..q1-1 whose positions fit the stage
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] - off[q0] <= St.cap) lo = mid; else hi = mid - 1;
    }
    const int q1 = lo, p0 = off[q0], np = off[q1] - p0;
    for (int x = threadIdx.x; x < np; x += blockDim.x) {
      int a = q0, z = q1 - 1;  // the route holding position p0 + x
      while (a < z) {
        const int mid = (a + z + 1) >> 1;
        if (off[mid] <= p0 + x) a = mid; else z = mid - 1;
      }
      const int p = p0 + x - off[a], n = off[a + 1] - off[a], r = list ? list[a] : a;
      const int *sq = P.seq + row_base(P, b, r);
      const int v = sq[p];
      if (p >= 1 && p <= n - (I.open ? 1 : 2)) {  // SolutionIndex entries of the customers
        LOC[v] = (r << 9) | (p - 1);
        NXS[v] = p + 1 <= n - 1 ? sq[p + 1] : -1;
      }
      const double2 *np2 = reinterpret_cast<const double2 *>(I.node + v);
      const double2 qs = __ldg(np2);
      St.load[x] = qs.x; St.T[x] = qs.y;
      if (WIN) { const double2 el = __ldg(np2 + 1); St.E[x] = el.x; St.L[x] = el.y; }
      St.v[x] = v;
      if (p > 0) { const Link lk = link_of(I, sq[p - 1], v); St.c[x] = lk.c; St.t[x] = lk.t; }
    }
    __syncthreads();
    RBT_(13);
    for (int q = q0 + gid; q < q1; q += ng) {
      const int r = list ? list[q] : q;
      const int4 mt = RM[r];
      const int n = off[q + 1] - off[q], base = off[q] - p0;
      for (int p = sub; p < (n + 1) / 2; p += kRbGroup) {
        fold_row_s<WIN>(I, P, b, r, St, base, p, n, mt);
        if (n - 1 - p != p) fold_row_s<WIN>(I, P, b, r, St, base, n - 1 - p, n, mt);
      }
    }
    __syncthreads();
    RBT_(14);
#ifdef MDR_SEL_PROF
    if (threadIdx.x == 0) atomicAdd(&g_selprof[15], 1ull);
#endif
    q0 = q1;
  }
}

// depot counts of non-empty routes -> fleet_inc/dec, excess (batch.py:144-158)
__device__ void rebuild_fleet(const DevInst &I, const DevPop &P, int b, int *sm_cnt) {
  const int m = P.m[b];
  const int4 *RM = P.rmeta + (size_t)b * P.J;
  for (int d = threadIdx.x; d < P.ND; d += blockDim.x) sm_cnt[d] = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    int4 mt = RM[r];
    if (mt.x > 0) atomicAdd(&sm_cnt[mt.y], 1);
  }
  __syncthreads();
  if (I.nv_on) {
    double2 *FL = P.fleet + (size_t)b * P.ND;
    for (int d = threadIdx.x; d < P.ND; d += blockDim.x) {
      double c = (double)sm_cnt[d];
      double over = npmax(c - I.NV, 0.0);
      FL[d] = make_double2(npmax((c + 1.0) - I.NV, 0.0) - over, npmax((c - 1.0) - I.NV, 0.0) - over);
    }
    if (threadIdx.x == 0) {
      double ex = 0.0;
      for (int d = 0; d < P.ND; d++) ex += npmax((double)sm_cnt[d] - I.NV, 0.0);
      P.fexcess[b] = ex;
    }
  } else if (threadIdx.x == 0) {
    P.fexcess[b] = 0.0;
  }
  __syncthreads();
}

// rebuild one individual (whole block): loc, tables, route terms, fleet
template <bool WIN>
__device__ void rebuild_block(const DevInst &I, const DevPop &P, int b, int *sm_cnt, int *off, int offcap, void *stg,
                              size_t stg_bytes) {
  int *LOC = P.loc + (size_t)b * P.N;
  for (int v = threadIdx.x; v < P.N; v += blockDim.x) { LOC[v] = -1; P.nxs[(size_t)b * P.N + v] = -1; }
  __syncthreads();
  rebuild_routes<WIN>(I, P, b, nullptr, P.m[b], off, offcap, stg, stg_bytes);
  __syncthreads();
  rebuild_fleet(I, P, b, sm_cnt);
}

template <bool WIN>
__global__ void __launch_bounds__(256) k_rebuild(DevInst I, DevPop P, int B) {
  extern __shared__ int sm_cnt[];  // [ND + 1], off [J + 1], staging (16-B aligned)
  int b = blockIdx.x;
  if (b >= B) return;
  int *off = sm_cnt + P.ND + 1;
  void *stg = reinterpret_cast<void *>((reinterpret_cast<uintptr_t>(off + P.J + 1) + 15) & ~uintptr_t(15));
  rebuild_block<WIN>(I, P, b, sm_cnt, off, P.J + 1, stg, kRbStageBytes);
}

// ---------------------------------------------------------------------------
// plan: operator of the round per individual, flattened chunk offsets
// ---------------------------------------------------------------------------
__device__ __forceinline__ int block_excl_scan(int x, int *wsum, int &total) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int inc = x;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, inc, s);
    if (lane >= s) inc += y;
  }
  __syncthreads();
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    int t = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, s);
      if (lane >= s) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  total = wsum[nw - 1];
  return inc - x + (w > 0 ? wsum[w - 1] : 0);
}

__global__ void __launch_bounds__(1024) k_plan(DevInst I, DevPop P, LsParams L) {
  // one pass: operator and task count of every active individual, appended to
  // its operator's list with one packed 64-bit shared atomic {index:24 | first task:40}
  // (list order is irrelevant: every result is reduced order-independently)
  __shared__ unsigned long long acc6[6];
  if (threadIdx.x < 6) acc6[threadIdx.x] = 0ull;
  __syncthreads();
  const unsigned long long MASK = (1ull << 40) - 1;
  for (int b = threadIdx.x; b < L.B; b += blockDim.x) {
    LsState st = P.st[b];
    P.fcount[b] = 0;
    P.nanflag[b] = 0;
    P.leader[b] = make_ulonglong2(~0ull, ~0ull);
    if (!st.done && st.pass >= P.maxp) {
      st.done = 1;
      st.status = 5;
      P.st[b] = st;
    }
    if (!st.done) {
      const int op = P.perms[((size_t)b * P.maxp + st.pass) * P.nops + st.pos];
      const int t = (P.staged && op <= 2) ? op_tasks_c(op, P.m[b], I.NC, P.ct) : op_tasks(op, P.m[b], I.NC, I.win);
      P.op_cur[b] = op;
      P.wsize[b] = t;
      if (t > 0) {
        unsigned long long old = atomicAdd(&acc6[op], (1ull << 40) | (unsigned long long)t);
        const int idx = (int)(old >> 40);
        P.opb[op * P.Bcap + idx] = b;
        P.opoff[op * (P.Bcap + 1) + idx] = (int)(old & MASK);
      }
    } else {
      P.op_cur[b] = -1;
      P.wsize[b] = 0;
    }
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int op = threadIdx.x;
    const int cnt = (int)(acc6[op] >> 40), tot = (int)(acc6[op] & MASK);
    P.opoff[op * (P.Bcap + 1) + cnt] = tot;
    P.opcnt[op] = cnt;
    P.optasks[op] = tot;
    P.task_next[op] = 0;
  }
  if (threadIdx.x == 0) {
    P.task_next[6] = 0;
    P.task_next[7] = 0;
    *P.active = 0;
    P.gcount[0] = 0;
    P.gcount[1] = 0;
    P.gcount[2] = 0;
  }
}

// ---------------------------------------------------------------------------
// fused enumerate + evaluate + reduce: persistent warps over the task list
// ---------------------------------------------------------------------------
#define MDR_TGRAB 2
#ifndef MDR_EVAL_MINB
#define MDR_EVAL_MINB 2
#endif

template <bool WIN, int OP>
__global__ void __launch_bounds__(256, MDR_EVAL_MINB) k_eval(DevInst I, DevPop P, LsParams L) {
  const int lane = threadIdx.x & 31;
  const int total = P.optasks[OP];
  const int cnt = P.opcnt[OP];
  const int *OFF = P.opoff + OP * (P.Bcap + 1);
  const int *OB = P.opb + OP * P.Bcap;
  const bool mm = L.multi_move != 0;
  __shared__ double s_u[8][MDR_USLOT];
  double *U = s_u[threadIdx.x >> 5];
  int lo = 0, hi = 0, b = 0;
  IV v;
  double lam[4] = {0, 0, 0, 0};
  for (;;) {
    int t0 = 0;
    if (lane == 0) t0 = atomicAdd(P.task_next + OP, MDR_TGRAB);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if (t0 >= total) break;
    const int t1 = min(t0 + MDR_TGRAB, total);
    for (int t = t0; t < t1; t++) {
      if (t < lo || t >= hi) {
        int l2 = 0, h2 = cnt - 1;  // last i with OFF[i] <= t
        while (l2 < h2) {
          int mid = (l2 + h2 + 1) >> 1;
          if (__ldg(OFF + mid) <= t) l2 = mid; else h2 = mid - 1;
        }
        b = OB[l2];
        lo = OFF[l2];
        hi = OFF[l2 + 1];
        v = make_iv(P, b);
#pragma unroll
        for (int i = 0; i < 4; i++) lam[i] = P.lam[b * 4 + i];
      }
      const int local = t - lo;
      Acc acc{~0ull, ~0ull, 0};
      if (OP == 0) task_relocate<WIN>(I, P, v, b, I.ND + local, lam, mm, acc, U);
      else if (OP == 1) task_swap<WIN>(I, P, v, b, I.ND + local, lam, mm, acc, U);
      else if (OP == 2) {
        if (local < I.NC) task_tos_u<WIN>(I, P, v, b, I.ND + local, lam, mm, acc);
        else task_tos_r<WIN>(I, P, v, b, local - I.NC, lam, mm, acc);
      } else if (OP == 3) task_two_opt<WIN>(I, P, v, b, I.ND + local, lam, mm, acc);
      else if (OP == 4) task_di<WIN>(I, P, v, b, local, lam, mm, acc);
      else task_dr<WIN>(I, P, v, b, local, lam, mm, acc);
      if (OP <= 2) {
        OK r = warp_min(OK{acc.o, acc.k});
        int n = acc.n;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) n += __shfl_xor_sync(0xffffffffu, n, s);
        if (lane == 0) {
          leader_min(P.leader + b, r.o, r.k);
          if (n) atomicAdd(&P.cands[(size_t)b * 6 + OP], (unsigned long long)n);
        }
      }
    }
  }
}

#ifndef MDR_WDMAX
#define MDR_WDMAX 32  // depot-indexed precomputes only up to this many depots
#endif
#ifndef MDR_TGC
#define MDR_TGC 1
#endif
#ifndef MDR_REL_WARP
#define MDR_REL_WARP 0  // 1: per-customer warp sweep (srelocate) instead of the flattened chunks
#endif
#ifndef MDR_SWAP_WARP
#define MDR_SWAP_WARP 0  // 1: per-customer warp sweep (sswap) instead of the flattened chunks
#endif
// CTA-task evaluators (relocate, swap, 2-opt*) with staged route boundaries
// FAM (relocate only): 0 both candidate families, 1 the granular (customer, list slot)
// items only, 2 the boundary (customer, route) items only -- two smaller kernels with
// their own register budgets
template <bool WIN, int OP, int CU, int CT, int MINB, int FAM = 0>
__global__ void __launch_bounds__(32 * CU, MINB) k_eval_c(DevInst I, DevPop P, LsParams L) {
  extern __shared__ __align__(16) unsigned char smx_c[];
  RBT<WIN> *R = reinterpret_cast<RBT<WIN> *>(smx_c);
  // per-warp depot-indexed precomputes (front-insertion prefixes, 2-opt* A sides)
  const int WS = I.ND <= MDR_WDMAX ? 18 * I.ND : 0;
  double *Wd = WS ? reinterpret_cast<double *>(smx_c + sizeof(RBT<WIN>) * P.J) + (threadIdx.x >> 5) * WS : nullptr;
  __shared__ double s_u[CU][MDR_USLOT];
  constexpr bool FLAT = OP == 1 && !MDR_SWAP_WARP;
  __shared__ __align__(16) double s_swd[FLAT ? CT * MDR_SWD : 1];
  __shared__ SWU s_sw[FLAT ? CT : 1];
  constexpr bool FLATR = OP == 0 && !MDR_REL_WARP;
  __shared__ __align__(16) double s_rld[FLATR ? CT * MDR_RLD : 1];
  __shared__ RLU s_rl[FLATR ? CT : 1];
  __shared__ int s_t, s_b, s_lo, s_hi, s_next, s_end;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *U = s_u[wid];
  // small populations: the relocate boundary family and the flattened swap split each
  // customer-block task into SPL sub-tasks (contiguous chunk ranges) for more CTAs per round
  const int SPL = ((OP == 0 && FAM == 2) || (OP == 1 && FLAT)) ? P.tsplit : 1;
  const int total = P.optasks[OP] * SPL;
  const int cnt = P.opcnt[OP];
  const int *OFF = P.opoff + OP * (P.Bcap + 1);
  const int *OB = P.opb + OP * P.Bcap;
  const bool mm = L.multi_move != 0;
  const int nch = (I.NC + CT - 1) / CT;
  __shared__ int s_item;
  int staged = -1;
  if (threadIdx.x == 0) { s_next = 0; s_end = 0; s_lo = 0; s_hi = 0; }
  for (;;) {
    if (threadIdx.x == 0) {
      // grab MDR_TGC consecutive tasks at a time: consecutive tasks belong to
      // the same individual, so its tables stay hot in this SM's L1
      if (s_next >= s_end) {
        int t0 = atomicAdd(P.task_next + (FAM == 2 ? 6 + OP : OP), MDR_TGC);
        s_next = t0;
        s_end = min(t0 + MDR_TGC, total);
      }
      int t = s_next < s_end ? s_next++ : total;
      s_t = t;
      s_item = 0;
      const int tb = t / SPL;  // the customer-block task
      if (t < total && (tb < s_lo || tb >= s_hi)) {
        int l2 = 0, h2 = cnt - 1;
        while (l2 < h2) {
          int mid = (l2 + h2 + 1) >> 1;
          if (OFF[mid] <= tb) l2 = mid; else h2 = mid - 1;
        }
        s_b = OB[l2];
        s_lo = OFF[l2];
        s_hi = OFF[l2 + 1];
      }
    }
    __syncthreads();
    const int t = s_t;
    if (t >= total) break;
    const int b = s_b, local = t / SPL - s_lo, sub = t - (t / SPL) * SPL;
    const IV v = make_iv(P, b);
    if (b != staged) {
      stage_routes<WIN>(I, v, R);
      staged = b;
    }
    __syncthreads();
    if (FLAT) {
      for (int j = threadIdx.x; j < CT; j += blockDim.x)
        sswap_stage<WIN>(I, v, R, I.ND + local * CT + j, s_sw[j], s_swd + j * MDR_SWD);
      __syncthreads();
    }
    if (FLATR) {
      for (int j = threadIdx.x; j < CT; j += blockDim.x)
        srel_stage<WIN>(I, v, R, I.ND + local * CT + j, s_rl[j], s_rld + j * MDR_RLD);
      __syncthreads();
    }
    double lam[4];
#pragma unroll
    for (int i = 0; i < 4; i++) lam[i] = P.lam[b * 4 + i];
    Acc acc{~0ull, ~0ull, 0};
    const int ngc = (CT * I.W + 31) / 32;
    const int ngb = (CT * v.M + 31) / 32;
    const int nall = FLAT ? ngc : FLATR ? (FAM == 1 ? ngc : FAM == 2 ? ngb : ngc + ngb) : CT;
    // sub-task `sub` of SPL owns chunks [c0, c1) of the customer-block task
    const int c0 = (int)((long long)nall * sub / SPL), c1 = (int)((long long)nall * (sub + 1) / SPL);
    const int nit = c1 - c0;
#ifndef MDR_ITEM_PREFETCH
#define MDR_ITEM_PREFETCH 1  // claim the next chunk while evaluating this one (C4 +0.7 %, C5 +0.8 %;
#endif                       // the same in k_eval_p measured -1 % at C5)
    int raw = 0;
    if (MDR_ITEM_PREFETCH && lane == 0) raw = atomicAdd(&s_item, 1);
    for (;;) {  // warps take the task's items dynamically
      int it = 0;
      if (MDR_ITEM_PREFETCH) {
        it = __shfl_sync(0xffffffffu, raw, 0);
        if (it >= nit) break;
        if (lane == 0) raw = atomicAdd(&s_item, 1);
      } else {
        if (lane == 0) it = atomicAdd(&s_item, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nit) break;
      }
      it += c0;
      if (FLATR) {
        if (FAM == 1) srel_chunk<WIN, CT>(I, P, v, R, b, it, false, s_rl, s_rld, lam, mm, acc);
        else if (FAM == 2) srel_chunk<WIN, CT>(I, P, v, R, b, it, true, s_rl, s_rld, lam, mm, acc);
        else srel_chunk<WIN, CT>(I, P, v, R, b, it < ngc ? it : it - ngc, it >= ngc, s_rl, s_rld, lam, mm, acc);
      } else if (FLAT) {
        sswap_chunk<WIN, CT, FAM>(I, P, v, R, b, it, s_sw, s_swd, lam, mm, acc);
      } else if (OP == 2 && local >= nch) {
        const int ra = (local - nch) * CT + it;
        if (ra < v.M) stos_r<WIN>(I, P, v, R, b, ra, lam, mm, acc);
      } else {
        const int u = I.ND + local * CT + it;
        if (u < I.N) {
          if (OP == 0) srelocate<WIN>(I, P, v, R, b, u, lam, mm, acc, U, Wd);
          else if (OP == 1) sswap<WIN>(I, P, v, R, b, u, lam, mm, acc, U);
          else stos_u<WIN>(I, P, v, R, b, u, lam, mm, acc, U, Wd);
        }
      }
    }
    OK r = warp_min(OK{acc.o, acc.k});
    int n = acc.n;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) n += __shfl_xor_sync(0xffffffffu, n, s);
    if (lane == 0) {
      leader_min(P.leader + b, r.o, r.k);
      if (n) atomicAdd(&P.cands[(size_t)b * 6 + OP], (unsigned long long)n);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Pipelined relocate / swap evaluators (the default for OP 0 and 1): the same
// flattened chunks as k_eval_c, but with no CTA-wide barrier.  Task staging is
// double-buffered -- two copies of the route boundaries and of the CT staged
// customers -- and handed over with mbarriers: the first warp to run out of
// items of task t fetches and stages task t+1 into the other buffer (one warp:
// routes strided over the lanes, one customer per lane) while the other warps
// finish task t; a warp releases a buffer (bar_free, one arrive per warp) when
// it is done with a task and waits on bar_ready before the next one.  The
// stager of a buffer waits for the release of its previous use, so no warp
// ever reads a buffer being rewritten.  Per task and warp the (dF, key) minimum
// and the candidate count are flushed to the individual as before.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long *bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long *bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

template <bool WIN>
__device__ __forceinline__ void stage_routes_warp(const DevInst &I, const IV &v, RBT<WIN> *R, int lane) {
  for (int r = lane; r < v.M; r += 32) {
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

// k_eval_p's stager: one warp fetches the next task and stages it into buffer nb
struct PipeShared {
  void *R0;  // RBT<WIN>[2][J]
  double *ud;  // [2][CT * UDW]
  void *cust;  // RLU[2][CT] or SWU[2][CT]
  unsigned long long *bar_ready, *bar_free;
  int *b, *local, *item, *first, *rbuf, *nst;
  int *next, *end, *lo, *hi, *bi;
};

template <bool WIN, int OP, int CT>
__device__ __forceinline__ void pipe_stage(const DevInst &I, const DevPop &P, const PipeShared &S, int nb) {
  constexpr int UDW = OP == 0 ? MDR_RLD : MDR_SWD;
  const int lane = threadIdx.x & 31;
  const int total = P.optasks[OP];
  const int cnt = P.opcnt[OP];
  const int *OFF = P.opoff + OP * (P.Bcap + 1);
  const int *OB = P.opb + OP * P.Bcap;
  const int nst = S.nst[nb];
  if (nst > 0) mb_wait(&S.bar_free[nb], (nst - 1) & 1);  // the previous use of nb is released
  if (lane == 0) {
    if (*S.next >= *S.end) {
      const int t0 = atomicAdd(P.task_next + OP, MDR_TGC);
      *S.next = t0;
      *S.end = min(t0 + MDR_TGC, total);
    }
    const int t = *S.next < *S.end ? (*S.next)++ : total;
    int b = -1;
    if (t < total) {
      if (t < *S.lo || t >= *S.hi) {
        int l2 = 0, h2 = cnt - 1;
        while (l2 < h2) {
          const int mid = (l2 + h2 + 1) >> 1;
          if (OFF[mid] <= t) l2 = mid; else h2 = mid - 1;
        }
        *S.bi = OB[l2];
        *S.lo = OFF[l2];
        *S.hi = OFF[l2 + 1];
      }
      b = *S.bi;
    }
    S.b[nb] = b;
    S.local[nb] = t - *S.lo;
    S.item[nb] = 0;
    S.first[nb] = 0;
  }
  __syncwarp();
  const int b = S.b[nb];
  if (b >= 0) {
    const IV v = make_iv(P, b);
    RBT<WIN> *R = reinterpret_cast<RBT<WIN> *>(S.R0) + (size_t)nb * P.J;
    if (S.rbuf[nb] != b) {
      stage_routes_warp<WIN>(I, v, R, lane);
      __syncwarp();
      if (lane == 0) S.rbuf[nb] = b;
    }
    const int u = I.ND + S.local[nb] * CT + lane;
    double *U = S.ud + ((size_t)nb * CT + lane) * UDW;
    if (lane < CT) {
      if (OP == 0) srel_stage<WIN>(I, v, R, u, reinterpret_cast<RLU *>(S.cust)[nb * CT + lane], U);
      else sswap_stage<WIN>(I, v, R, u, reinterpret_cast<SWU *>(S.cust)[nb * CT + lane], U);
    }
  }
  __syncwarp();
  __threadfence_block();
  if (lane == 0) {
    S.nst[nb] = nst + 1;
    mb_arrive(&S.bar_ready[nb]);
  }
}

template <bool WIN, int OP, int CU, int CT, int MINB>
__global__ void __launch_bounds__(32 * CU, MINB) k_eval_p(DevInst I, DevPop P, LsParams L) {
  static_assert(OP == 0 || OP == 1, "pipelined form: relocate and swap");
  static_assert(CT <= 32, "one staged customer per lane");
  extern __shared__ __align__(16) unsigned char smx_c[];
  RBT<WIN> *const R0 = reinterpret_cast<RBT<WIN> *>(smx_c);
  constexpr int UDW = OP == 0 ? MDR_RLD : MDR_SWD;
  __shared__ __align__(16) double s_ud[2][CT * UDW];
  __shared__ RLU s_rl[OP == 0 ? 2 : 1][OP == 0 ? CT : 1];
  __shared__ SWU s_sw[OP == 1 ? 2 : 1][OP == 1 ? CT : 1];
  __shared__ __align__(8) unsigned long long bar_ready[2], bar_free[2];
  __shared__ int s_b[2], s_local[2], s_item[2], s_first[2], s_rbuf[2], s_nst[2];
  __shared__ int s_next, s_end, s_lo, s_hi, s_bi;
  const int lane = threadIdx.x & 31;
  const bool mm = L.multi_move != 0;
  if (threadIdx.x == 0) {
    mb_init(&bar_ready[0], 1);
    mb_init(&bar_ready[1], 1);
    mb_init(&bar_free[0], CU);
    mb_init(&bar_free[1], CU);
    s_next = 0; s_end = 0; s_lo = 0; s_hi = 0; s_bi = -1;
    s_rbuf[0] = s_rbuf[1] = -1;
    s_nst[0] = s_nst[1] = 0;
  }
  __syncthreads();
  PipeShared S;
  S.R0 = R0;
  S.ud = &s_ud[0][0];
  S.cust = OP == 0 ? (void *)&s_rl[0][0] : (void *)&s_sw[0][0];
  S.bar_ready = bar_ready; S.bar_free = bar_free;
  S.b = s_b; S.local = s_local; S.item = s_item; S.first = s_first; S.rbuf = s_rbuf; S.nst = s_nst;
  S.next = &s_next; S.end = &s_end; S.lo = &s_lo; S.hi = &s_hi; S.bi = &s_bi;
  if ((threadIdx.x >> 5) == 0) pipe_stage<WIN, OP, CT>(I, P, S, 0);
  int buf = 0;
  unsigned use[2] = {0u, 0u};
  for (;;) {
    mb_wait(&bar_ready[buf], use[buf] & 1);
    const int b = s_b[buf];
    if (b < 0) break;
    const IV v = make_iv(P, b);
    const RBT<WIN> *R = R0 + (size_t)buf * P.J;
    double lam[4];
#pragma unroll
    for (int i = 0; i < 4; i++) lam[i] = P.lam[b * 4 + i];
    Acc acc{~0ull, ~0ull, 0};
    const int ngc = (CT * I.W + 31) / 32;
    const int nit = OP == 1 ? ngc : ngc + (CT * v.M + 31) / 32;
    for (;;) {
      int it = 0;
      if (lane == 0) it = atomicAdd(&s_item[buf], 1);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= nit) break;
      if (OP == 0)
        srel_chunk<WIN, CT>(I, P, v, R, b, it < ngc ? it : it - ngc, it >= ngc, s_rl[OP == 0 ? buf : 0], s_ud[buf],
                            lam, mm, acc);
      else
        sswap_chunk<WIN, CT>(I, P, v, R, b, it, s_sw[OP == 1 ? buf : 0], s_ud[buf], lam, mm, acc);
    }
    OK r = warp_min(OK{acc.o, acc.k});
    int n = acc.n;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) n += __shfl_xor_sync(0xffffffffu, n, s);
    int first = 0;
    __syncwarp();
    if (lane == 0) {
      leader_min(P.leader + b, r.o, r.k);
      if (n) atomicAdd(&P.cands[(size_t)b * 6 + OP], (unsigned long long)n);
      first = atomicAdd(&s_first[buf], 1) == 0;
      mb_arrive(&bar_free[buf]);
    }
    first = __shfl_sync(0xffffffffu, first, 0);
    use[buf]++;
    if (first) pipe_stage<WIN, OP, CT>(I, P, S, buf ^ 1);
    buf ^= 1;
  }
}

// generic evaluator: intra-route relocate/swap, 2-opt, depot operators,
// one thread per queued candidate through eval_cand (batch.py:365-553).
// FOP 0 / 1: the per-producer regions 1 / 2, which hold only same-route
// relocate / swap candidates; -1: any operator (region 0, single queue).
template <bool WIN, int FOP>
#ifndef MDR_GMINB
#define MDR_GMINB 3
#endif
#ifndef MDR_GMINB_I
#define MDR_GMINB_I 2  // the same-route forms hold a whole candidate's loads at once
#endif
__global__ void __launch_bounds__(256, FOP >= 0 ? MDR_GMINB_I : MDR_GMINB) k_eval_g(DevInst I, DevPop P, LsParams L, int region) {
  const int lane = threadIdx.x & 31;
  const int total = min(P.gcount[region], P.gbase[region + 1] - P.gbase[region]);
  const ulonglong2 *Q = P.gq + P.gbase[region];
  const bool mm = L.multi_move != 0;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  // the next batch's queue entry is loaded one iteration ahead (it heads the
  // dependent load chain entry -> route meta -> table rows)
#ifndef MDR_G_PREFETCH
#define MDR_G_PREFETCH 1
#endif
  ulonglong2 nx = make_ulonglong2(0ull, 0ull);
  if (MDR_G_PREFETCH && wid * 32 + lane < total) nx = Q[wid * 32 + lane];
  for (int base = wid * 32; base < total; base += nwarps * 32) {
    const int i = base + lane;
    const bool valid = i < total;
    ulonglong2 e = nx;
    if (!MDR_G_PREFETCH) e = valid ? Q[i] : make_ulonglong2(0ull, 0ull);
    else if (i + nwarps * 32 < total) nx = Q[i + nwarps * 32];
    int b = -1, op = 0;
    unsigned long long key = 0, o = ~0ull;
    bool fol = false;
    if (valid) {
      key = e.x;
      b = (int)(e.y & 0xffffffu);
      op = (int)(e.y >> 24);
      double lam[4];
#pragma unroll
      for (int q = 0; q < 4; q++) lam[q] = P.lam[b * 4 + q];
      Delta D;
      if constexpr (FOP >= 0) D = eval_intra<WIN, FOP>(I, P, b, unpack_key(key), lam);
      else D = eval_cand<WIN>(I, P, b, op, unpack_key(key), lam);
      if (D.dF != D.dF) {
        atomicOr(P.nanflag + b, 1);
      } else {
        o = ord_of(D.dF);
        fol = mm && follower_ok(D);
      }
    }
    const int b0 = __shfl_sync(0xffffffffu, b, 0);
    const bool uni = __all_sync(0xffffffffu, !valid || b == b0);
    if (uni) {
      OK r = warp_min(OK{o, key});
      unsigned vm = __ballot_sync(0xffffffffu, valid);
      const int op0 = __shfl_sync(0xffffffffu, op, 0);
      if (lane == 0) {
        leader_min(P.leader + b0, r.o, r.k);
        atomicAdd(&P.cands[(size_t)b0 * 6 + op0], (unsigned long long)__popc(vm));
      }
      append_fol(P, b0, fol, o, key);
    } else if (valid) {
      leader_min(P.leader + b, o, key);
      atomicAdd(&P.cands[(size_t)b * 6 + op], 1ull);
      if (fol) {
        int at = atomicAdd(&P.fcount[b], 1);
        if (at < P.Fcap) P.fol[(size_t)b * P.Fcap + at] = make_ulonglong2(o, key);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// select + apply + rebuild + adapt
// ---------------------------------------------------------------------------
__device__ __forceinline__ void put_range(int *dst, int &k, const int *src, int from, int to) {
  for (int i = from; i < to; i++) dst[1 + k++] = src[1 + i];
}

// one move (route-disjoint from the others of the round); reads old rows
// from scratch, writes the live rows (moves.move_plan, moves.py:88-148)
__device__ bool apply_one(const DevInst &I, const DevPop &P, int b, int op, const Cand &c, int new_r) {
  const int *S1 = P.scratch_seq + row_base(P, b, c.r1);
  const int4 M1 = P.scratch_meta[(size_t)b * P.J + c.r1];
  int *D1 = P.seq + row_base(P, b, c.r1);
  int4 *RM = P.rmeta + (size_t)b * P.J;
  const int K = P.K;
  int k1 = M1.x;
  int seg[2];
  auto finish = [&](int *row, int r, int dep, int arr, int k) -> bool {
    if (k > K) return false;
    row[0] = dep;
    if (!I.open) row[k + 1] = arr;
    RM[r] = make_int4(k, dep, arr, 0);
    return true;
  };
  switch (op) {
    case 0: {
      for (int i = 0; i < c.l1; i++) seg[i] = S1[1 + c.p1 + i];
      if (c.rev1 && c.l1 == 2) { int t = seg[0]; seg[0] = seg[1]; seg[1] = t; }
      if (c.r1 == c.r2) {
        int at = c.p2 > c.p1 ? c.p2 - c.l1 : c.p2;
        int k = 0, ri = 0;  // ri indexes "rest" = customers without the segment
        for (int i = 0; i < k1 && k <= K; i++) {
          if (i >= c.p1 && i < c.p1 + c.l1) continue;
          if (ri == at) for (int s = 0; s < c.l1; s++) D1[1 + k++] = seg[s];
          D1[1 + k++] = S1[1 + i];
          ri++;
        }
        if (ri == at) for (int s = 0; s < c.l1; s++) D1[1 + k++] = seg[s];
        return finish(D1, c.r1, M1.y, M1.z, k);
      }
      const int *S2 = P.scratch_seq + row_base(P, b, c.r2);
      const int4 M2 = P.scratch_meta[(size_t)b * P.J + c.r2];
      int *D2 = P.seq + row_base(P, b, c.r2);
      int ka = 0;
      put_range(D1, ka, S1, 0, c.p1);
      put_range(D1, ka, S1, c.p1 + c.l1, k1);
      if (!finish(D1, c.r1, M1.y, M1.z, ka)) return false;
      if (M2.x + c.l1 > K) return false;
      int kb = 0;
      put_range(D2, kb, S2, 0, c.p2);
      for (int s = 0; s < c.l1; s++) D2[1 + kb++] = seg[s];
      put_range(D2, kb, S2, c.p2, M2.x);
      return finish(D2, c.r2, M2.y, M2.z, kb);
    }
    case 1: {
      int s1[2], s2[2];
      const int *S2 = c.r1 == c.r2 ? S1 : P.scratch_seq + row_base(P, b, c.r2);
      const int4 M2 = c.r1 == c.r2 ? M1 : P.scratch_meta[(size_t)b * P.J + c.r2];
      for (int i = 0; i < c.l1; i++) s1[i] = S1[1 + c.p1 + i];
      if (c.rev1 && c.l1 == 2) { int t = s1[0]; s1[0] = s1[1]; s1[1] = t; }
      for (int i = 0; i < c.l2; i++) s2[i] = S2[1 + c.p2 + i];
      if (c.rev2 && c.l2 == 2) { int t = s2[0]; s2[0] = s2[1]; s2[1] = t; }
      if (c.r1 == c.r2) {
        int k = 0;
        put_range(D1, k, S1, 0, c.p1);
        for (int s = 0; s < c.l2; s++) D1[1 + k++] = s2[s];
        put_range(D1, k, S1, c.p1 + c.l1, c.p2);
        for (int s = 0; s < c.l1; s++) D1[1 + k++] = s1[s];
        put_range(D1, k, S1, c.p2 + c.l2, k1);
        return finish(D1, c.r1, M1.y, M1.z, k);
      }
      if (k1 - c.l1 + c.l2 > K || M2.x - c.l2 + c.l1 > K) return false;
      int *D2 = P.seq + row_base(P, b, c.r2);
      int ka = 0, kb = 0;
      put_range(D1, ka, S1, 0, c.p1);
      for (int s = 0; s < c.l2; s++) D1[1 + ka++] = s2[s];
      put_range(D1, ka, S1, c.p1 + c.l1, k1);
      put_range(D2, kb, S2, 0, c.p2);
      for (int s = 0; s < c.l1; s++) D2[1 + kb++] = s1[s];
      put_range(D2, kb, S2, c.p2 + c.l2, M2.x);
      return finish(D1, c.r1, M1.y, M1.z, ka) && finish(D2, c.r2, M2.y, M2.z, kb);
    }
    case 3: {
      int k = 0;
      put_range(D1, k, S1, 0, c.p1);
      for (int i = c.p2; i >= c.p1; i--) D1[1 + k++] = S1[1 + i];
      put_range(D1, k, S1, c.p2 + 1, k1);
      return finish(D1, c.r1, M1.y, M1.z, k);
    }
    case 2: {
      const int *S2 = P.scratch_seq + row_base(P, b, c.r2);
      const int4 M2 = P.scratch_meta[(size_t)b * P.J + c.r2];
      int *D2 = P.seq + row_base(P, b, c.r2);
      int ka = c.p1 + (M2.x - c.p2), kb = c.p2 + (k1 - c.p1);
      if (ka > K || kb > K) return false;
      ka = 0; kb = 0;
      put_range(D1, ka, S1, 0, c.p1);
      put_range(D1, ka, S2, c.p2, M2.x);
      put_range(D2, kb, S2, 0, c.p2);
      put_range(D2, kb, S1, c.p1, k1);
      return finish(D1, c.r1, M1.y, M2.z, ka) && finish(D2, c.r2, M2.y, M1.z, kb);
    }
    case 4: {
      if (new_r >= P.J) return false;
      int *DN = P.seq + row_base(P, b, new_r);
      int ka = 0, kn = 0;
      put_range(DN, kn, S1, c.p1, k1);
      put_range(D1, ka, S1, 0, c.p1);
      return finish(D1, c.r1, M1.y, M1.z, ka) && finish(DN, new_r, c.depot, c.depot, kn);
    }
    default: {
      int dep = (c.mode == 0 || c.mode == 2) ? c.depot : M1.y;
      int arr = (c.mode == 1 || c.mode == 2) ? c.depot : M1.z;
      int k = 0;
      put_range(D1, k, S1, 0, k1);
      return finish(D1, c.r1, dep, arr, k);
    }
  }
}

#ifdef MDR_SEL_PROF
#define SELT(i) do { if (threadIdx.x == 0) { long long t__ = clock64(); atomicAdd(&g_selprof[i], (unsigned long long)(t__ - t_sel)); t_sel = t__; } } while (0)
#else
#define SELT(i) do { } while (0)
#endif
#ifndef MDR_SEL_WARP
#define MDR_SEL_WARP 1  // 0: repeated block argmin for fewer than 256 followers too
#endif
constexpr int kSelWarpFw = 8;  // followers per lane of the warp selection

#ifndef MDR_TOS_W_MINB
#define MDR_TOS_W_MINB 3  // 2-opt* with windows: 8-warp CTAs, this many per SM
#endif
#ifndef MDR_TOS_NW_SHAPE
#define MDR_TOS_NW_SHAPE 0  // 2-opt* without windows: 0 = 16 warps x 128, 1 = 24 x 80
#endif
#ifndef MDR_REL_NW_SHAPE
#define MDR_REL_NW_SHAPE 0  // relocate without windows: 0 = 20 warps x 96, 1 = 24 x 80
#endif
#ifndef MDR_SWAP_SHAPE_DEFAULT
#define MDR_SWAP_SHAPE_DEFAULT 1  // 20 warps x 96 with the u-side-outer swap: C4 +2.4 % over the pipelined 16 x 128
#endif
#ifndef MDR_SEL_SORT
#define MDR_SEL_SORT 2048  // followers sorted in shared memory up to this many (else repeated block argmin)
#endif
constexpr size_t kSelStageBytes =
    sizeof(ulonglong2) * MDR_SEL_SORT > kRbStageBytes ? sizeof(ulonglong2) * MDR_SEL_SORT : kRbStageBytes;

#ifndef MDR_SEL_THREADS
#define MDR_SEL_THREADS 512  // one CTA per individual: more warps rebuild more touched routes at once
#endif
template <bool WIN>
__global__ void __launch_bounds__(MDR_SEL_THREADS, 1) k_select(DevInst I, DevPop P, LsParams L) {
  extern __shared__ unsigned long long smx[];
  __shared__ OK red[MDR_SEL_THREADS / 32];
  __shared__ int s_flag, s_nm, s_mnew, s_snap, s_nt, s_empty, s_feas;
  __shared__ double s_D;
  __shared__ unsigned long long s_leader;
  const int b = blockIdx.x;
  if (b >= L.B) return;
  if (P.st[b].done) return;
#ifdef MDR_SEL_PROF
  long long t_sel = clock64();
  const long long t_sel0 = t_sel;
  if (threadIdx.x == 0) atomicAdd(&g_selprof[8], 1ull);  // active CTA-rounds
#endif
  const int J = P.J;
  unsigned long long *sel = smx;                            // [J] selected keys
  unsigned *used = reinterpret_cast<unsigned *>(sel + J);   // [J/32+1] route bitmask
  int *newidx = reinterpret_cast<int *>(used + (J / 32 + 1));  // [J+J]
  int *sm_cnt = newidx + 2 * J;                             // [ND]
  int *tl = sm_cnt + P.ND + 4;                              // [3J] touched routes
  // sorted followers (select phase) / staged route positions (rebuild phase)
  void *stg = reinterpret_cast<void *>((reinterpret_cast<uintptr_t>(tl + 3 * J + 1) + 15) & ~uintptr_t(15));
  const size_t stg_bytes = kSelStageBytes;
  const int op = P.op_cur[b];

  // ---- leader (batch.py:587-597): the round's min (dF, key) of this individual
  const ulonglong2 ld = P.leader[b];
  const OK best{ld.x, ld.y};
  const bool has = !P.nanflag[b] && best.o != ~0ull && unord(best.o) < -MDR_EPS;
  const int nf = P.fcount[b];
  if (threadIdx.x == 0) {
    P.st[b].op_evals++;
    s_flag = 0;
    if (has && L.multi_move && nf > P.Fcap) { s_flag = 1; P.st[b].need_f = nf; }  // follower buffer overflow
    int gneed = 0;  // generic queue overflow: the region sizes scale with Gcap
    for (int r = 0; r < 3; r++) {
      const int cap = P.gbase[r + 1] - P.gbase[r];
      if (P.gcount[r] > cap) gneed = max(gneed, (int)((long long)P.gcount[r] * P.Gcap / max(cap, 1)) + 1);
    }
    if (gneed) { s_flag = 1; P.st[b].need_g = gneed; }
  }
  __syncthreads();
  if (s_flag) {
    if (threadIdx.x == 0) { P.st[b].done = 1; P.st[b].status = 3; }
    return;
  }
  if (has) {
    // ---- select_moves (localsearch.py:45-55): greedy in (dF, key) order ==
    // repeated argmin over followers not touching used routes
    for (int i = threadIdx.x; i < J / 32 + 1; i += blockDim.x) used[i] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
      s_leader = best.k;
      sel[0] = best.k;
      Cand c = unpack_key(best.k);
      used[c.r1 >> 5] |= 1u << (c.r1 & 31);
      if (c.r2 >= 0) used[c.r2 >> 5] |= 1u << (c.r2 & 31);
      s_nm = 1;
    }
    __syncthreads();
    if (L.multi_move && nf >= 256 && nf <= MDR_SEL_SORT) {
      // followers sorted once by (dF, key) in shared memory (bitonic), then one
      // warp walks them in order 32 at a time: the lowest lane whose move touches
      // no used route is taken, the others re-check -- the greedy of
      // select_moves without a block-wide argmin per selected move
      const ulonglong2 *F = P.fol + (size_t)b * P.Fcap;
      ulonglong2 *S = reinterpret_cast<ulonglong2 *>(stg);
      int n2 = 32;
      while (n2 < nf) n2 <<= 1;
      for (int i = threadIdx.x; i < n2; i += blockDim.x)
        S[i] = i < nf && F[i].y != s_leader ? F[i] : make_ulonglong2(~0ull, ~0ull);
      __syncthreads();
      for (int kk = 2; kk <= n2; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          for (int i = threadIdx.x; i < n2; i += blockDim.x) {
            const int l = i ^ jj;
            if (l > i) {
              const ulonglong2 a = S[i], c = S[l];
              const bool gt = a.x > c.x || (a.x == c.x && a.y > c.y);
              if (gt == ((i & kk) == 0)) { S[i] = c; S[l] = a; }
            }
          }
          __syncthreads();
        }
      }
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int nm = s_nm;
        for (int base = 0; base < nf; base += 32) {
          const ulonglong2 e = S[base + lane];
          const bool valid = e.x != ~0ull;
          Cand c = unpack_key(e.y);
          bool taken = false;
          if (!__any_sync(0xffffffffu, valid)) break;
          for (;;) {
            bool ok = valid && !taken && !((used[c.r1 >> 5] >> (c.r1 & 31)) & 1u);
            if (ok && c.r2 >= 0) ok = !((used[c.r2 >> 5] >> (c.r2 & 31)) & 1u);
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            if (!m) break;
            const int w = __ffs(m) - 1;
            if (lane == w) {
              taken = true;
              sel[nm] = e.y;
              used[c.r1 >> 5] |= 1u << (c.r1 & 31);
              if (c.r2 >= 0) used[c.r2 >> 5] |= 1u << (c.r2 & 31);
            }
            nm++;
            __syncwarp();
          }
        }
        if (lane == 0) s_nm = nm;
      }
      __syncthreads();
    } else if (L.multi_move && nf <= 32 * kSelWarpFw && MDR_SEL_WARP) {
      // up to 32 * kSelWarpFw followers: one warp holds them in registers and
      // repeats a warp argmin over the non-conflicting ones (no CTA barriers)
      if (threadIdx.x < 32) {
        const ulonglong2 *F = P.fol + (size_t)b * P.Fcap;
        const int lane = threadIdx.x;
        unsigned long long eo[kSelWarpFw], ek[kSelWarpFw];
        int e1[kSelWarpFw], e2[kSelWarpFw];
#pragma unroll
        for (int q = 0; q < kSelWarpFw; q++) {
          const int i = lane + 32 * q;
          eo[q] = ~0ull; ek[q] = ~0ull; e1[q] = 0; e2[q] = -1;
          if (i < nf) {
            const ulonglong2 e = F[i];
            if (e.y != s_leader) {
              const Cand c = unpack_key(e.y);
              eo[q] = e.x; ek[q] = e.y; e1[q] = c.r1; e2[q] = c.r2;
            }
          }
        }
        int nm = s_nm;
        for (;;) {
          OK x{~0ull, ~0ull};
#pragma unroll
          for (int q = 0; q < kSelWarpFw; q++) {
            bool conflict = (used[e1[q] >> 5] >> (e1[q] & 31)) & 1u;
            if (e2[q] >= 0) conflict = conflict || ((used[e2[q] >> 5] >> (e2[q] & 31)) & 1u);
            const OK y{eo[q], ek[q]};
            if (eo[q] != ~0ull && !conflict && ok_less(y, x)) x = y;
          }
          x = warp_min(x);
          if (x.o == ~0ull) break;
          __syncwarp();
          if (lane == 0) {
            sel[nm] = x.k;
            const Cand c = unpack_key(x.k);
            used[c.r1 >> 5] |= 1u << (c.r1 & 31);
            if (c.r2 >= 0) used[c.r2 >> 5] |= 1u << (c.r2 & 31);
          }
          nm++;
          __syncwarp();
        }
        if (lane == 0) s_nm = nm;
      }
      __syncthreads();
    } else if (L.multi_move) {
      const ulonglong2 *F = P.fol + (size_t)b * P.Fcap;
      for (;;) {
        OK x{~0ull, ~0ull};
        for (int i = threadIdx.x; i < nf; i += blockDim.x) {
          ulonglong2 e = F[i];
          if (e.y == s_leader) continue;
          Cand c = unpack_key(e.y);
          bool conflict = (used[c.r1 >> 5] >> (c.r1 & 31)) & 1u;
          if (c.r2 >= 0) conflict = conflict || ((used[c.r2 >> 5] >> (c.r2 & 31)) & 1u);
          OK y{e.x, e.y};
          if (!conflict && ok_less(y, x)) x = y;
        }
        x = block_min(x, red);
        if (x.o == ~0ull) break;
        if (threadIdx.x == 0) {
          sel[s_nm++] = x.k;
          Cand c = unpack_key(x.k);
          used[c.r1 >> 5] |= 1u << (c.r1 & 31);
          if (c.r2 >= 0) used[c.r2 >> 5] |= 1u << (c.r2 & 31);
        }
        __syncthreads();
      }
    }
    SELT(0);  // leader + follower selection
    // ---- apply_moves (localsearch.py:58-82); touched routes staged in scratch
    const int m = P.m[b];
    const int nm = s_nm;
    if (threadIdx.x == 0) {
      int nt = 0;
      for (int t = 0; t < nm; t++) {
        Cand c = unpack_key(sel[t]);
        tl[nt++] = c.r1;
        if (c.r2 >= 0 && c.r2 != c.r1) tl[nt++] = c.r2;
      }
      s_nt = nt;
      s_flag = 0;
    }
    __syncthreads();
    {  // warp per touched route, its k+2 used sequence slots
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int q = wid; q < s_nt; q += nw) {
        const int r = tl[q], len = P.rmeta[(size_t)b * J + r].x + 2;
        for (int x = lane; x < len; x += 32) P.scratch_seq[row_base(P, b, r) + x] = P.seq[row_base(P, b, r) + x];
      }
    }
    for (int i = threadIdx.x; i < s_nt; i += blockDim.x)
      P.scratch_meta[(size_t)b * J + tl[i]] = P.rmeta[(size_t)b * J + tl[i]];
    __syncthreads();
    for (int t = threadIdx.x; t < nm; t += blockDim.x) {
      Cand c = unpack_key(sel[t]);
      if (!apply_one(I, P, b, op, c, m + t)) {
        s_flag = 1;
        atomicMax(&P.st[b].need_j, m + nm);
        atomicMax(&P.st[b].need_k, 2 * P.K);
      }
    }
    __syncthreads();
    if (s_flag) {
      if (threadIdx.x == 0) { P.st[b].done = 1; P.st[b].status = 3; }
      return;
    }
    SELT(1);  // apply
    // drop_empty_routes (model.py:198-199), stable; DI tails were appended at m+t
    const int m2 = m + (op == 4 ? nm : 0);
    // drop_empty_routes removes every empty route, including ones the input carried
    if (threadIdx.x == 0) s_empty = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < m; r += blockDim.x)
      if (P.rmeta[(size_t)b * J + r].x == 0) s_empty = 1;
    __syncthreads();
    if (!s_empty) {
      // no index shifts: only the touched routes and the appended depot-insert
      // tails change; their tables, terms and SolutionIndex entries are rebuilt
      if (threadIdx.x == 0) {
        int nt = s_nt;
        for (int r = m; r < m2; r++) tl[nt++] = r;
        s_nt = nt;
        P.m[b] = m2;
        s_mnew = m2;
      }
      __syncthreads();
      rebuild_routes<WIN>(I, P, b, tl, s_nt, newidx, 2 * J, stg, stg_bytes);
      __syncthreads();
      SELT(2);  // incremental rebuild
      rebuild_fleet(I, P, b, sm_cnt);
    } else {
    // drop the empty routes: lengths loaded by all threads at once, one warp
    // scans keep flags and kept lengths in shared memory, then the sequences
    // move position-parallel through the scratch rows
    int *klen = tl, *oldof = tl + J, *off2 = tl + 2 * J;  // [J], [J], [J + 1] (tl has 3J + 1)
    for (int r = threadIdx.x; r < m2; r += blockDim.x) klen[r] = P.rmeta[(size_t)b * J + r].x;
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int carry = 0, pos = 0;
      for (int base = 0; base < m2; base += 32) {
        const int r = base + lane;
        const bool keep = r < m2 && klen[r] > 0;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        const int ni = carry + __popc(bal & ((1u << lane) - 1));
        int x = keep ? klen[r] + 2 : 0;  // the k+2 used sequence slots
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, d);
          if (lane >= d) x += y;
        }
        if (keep) { oldof[ni] = r; off2[ni + 1] = pos + x; }
        pos += __shfl_sync(0xffffffffu, x, 31);
        carry += __popc(bal);
      }
      if (lane == 0) { s_mnew = carry; off2[0] = 0; }
    }
    __syncthreads();
    const int mn_ = s_mnew, tot = off2[mn_];
    for (int x = threadIdx.x; x < tot; x += blockDim.x) {
      int a = 0, z = mn_ - 1;
      while (a < z) {
        const int mid = (a + z + 1) >> 1;
        if (off2[mid] <= x) a = mid; else z = mid - 1;
      }
      const int p = x - off2[a];
      P.scratch_seq[row_base(P, b, a) + p] = P.seq[row_base(P, b, oldof[a]) + p];
    }
    for (int q = threadIdx.x; q < mn_; q += blockDim.x)
      P.scratch_meta[(size_t)b * J + q] = P.rmeta[(size_t)b * J + oldof[q]];
    __syncthreads();
    for (int x = threadIdx.x; x < tot; x += blockDim.x) {
      int a = 0, z = mn_ - 1;
      while (a < z) {
        const int mid = (a + z + 1) >> 1;
        if (off2[mid] <= x) a = mid; else z = mid - 1;
      }
      const int p = x - off2[a];
      P.seq[row_base(P, b, a) + p] = P.scratch_seq[row_base(P, b, a) + p];
    }
    for (int q = threadIdx.x; q < mn_; q += blockDim.x) P.rmeta[(size_t)b * J + q] = P.scratch_meta[(size_t)b * J + q];
    if (threadIdx.x == 0) P.m[b] = mn_;
    __syncthreads();
#ifdef MDR_SEL_PROF
    if (threadIdx.x == 0) atomicAdd(&g_selprof[11], (unsigned long long)(clock64() - t_sel));
#endif
    rebuild_block<WIN>(I, P, b, sm_cnt, newidx, 2 * J, stg, stg_bytes);
    SELT(3);  // full rebuild (a route emptied)
#ifdef MDR_SEL_PROF
    if (threadIdx.x == 0) atomicAdd(&g_selprof[9], 1ull);
#endif
    }
    const int mn = s_mnew;
    SELT(4);  // fleet (incremental path)
    // ---- totals, adapt_penalties, bookkeeping (localsearch.py:128-138)
    // the four pairwise sums run on four warps; the closure count (0/1 values,
    // exact in any order) on a fifth
    __shared__ double s_tot[5];
    {
      const int wid = threadIdx.x >> 5;
      const double4 *RC = P.rcon + (size_t)b * J;
      if ((threadIdx.x & 31) == 0) {
        if (wid < 4) s_tot[wid] = pw_sum(RC, wid, mn);
        else if (wid == 4) {
          double clo = 0.0;
          for (int r = 0; r < mn; r++) clo += (double)P.rmeta[(size_t)b * J + r].w;
          s_tot[4] = I.theta * (clo + P.fexcess[b]);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot[5] = {s_tot[0], s_tot[1], s_tot[2], s_tot[3], s_tot[4]};
      LsState st = P.st[b];
      bool feas = true;
      for (int i = 0; i < 4; i++) {
        double lm = P.lam[b * 4 + i];
        bool viol = tot[i + 1] > 1e-9;
        if (viol) { lm = lm / L.kappa; feas = false; }
        else lm = lm * L.kappa;
        double x = L.lam_min > lm ? L.lam_min : lm;
        P.lam[b * 4 + i] = L.lam_max < x ? L.lam_max : x;
      }
      s_snap = 0;
      s_feas = feas;
      s_D = tot[0];
      if (feas) {
        st.n_feasible++;
        if (tot[0] < st.bestD) { st.bestD = tot[0]; st.n_improving++; s_snap = L.snapshot; }
      }
      st.accepted++;
      st.any = 1;
      st.moves_applied += nm;
      if (st.accepted >= L.depth) st.done = 1;
      P.st[b] = st;
    }
    __syncthreads();
    if (L.trace) {  // the accepted step for the host's per-state on_feasible replay
      const long long at = P.trcount[b];
      unsigned long long *T = P.trace + (size_t)b * P.tcap + at;
      if (at + 2 + nm <= P.tcap) {
        for (int t = threadIdx.x; t < nm; t += blockDim.x) T[2 + t] = sel[t];
        if (threadIdx.x == 0) {
          T[0] = ((unsigned long long)op << 56) | ((unsigned long long)(s_feas ? 1 : 0) << 55) | (unsigned)nm;
          T[1] = (unsigned long long)__double_as_longlong(s_D);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) P.trcount[b] = at + 2 + nm;  // past tcap: overflow, reported by the host
    }
    if (s_snap) {  // best-feasible snapshot, only when the caller wants it (on_feasible)
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int r = wid; r < mn; r += nw) {
        const int len = P.rmeta[(size_t)b * J + r].x + 2;
        for (int x = lane; x < len; x += 32) P.best_seq[row_base(P, b, r) + x] = P.seq[row_base(P, b, r) + x];
      }
      for (int r = threadIdx.x; r < mn; r += blockDim.x)
        P.best_meta[(size_t)b * J + r] = P.rmeta[(size_t)b * J + r];
      if (threadIdx.x == 0) P.best_m[b] = mn;
    }
  }
  SELT(5);  // totals, adapt, trace, snapshot
#ifdef MDR_SEL_PROF
  if (threadIdx.x == 0) atomicMax(&g_selprof[10], (unsigned long long)(t_sel - t_sel0));
#endif
  // ---- advance the pass/operator cursor
  if (threadIdx.x == 0) {
    LsState st = P.st[b];
    if (!st.done) {
      st.pos++;
      if (st.pos >= P.nops) {
        if (!st.any) st.done = 1;
        else { st.pass++; st.pos = 0; st.any = 0; }
      }
      P.st[b] = st;
    }
    if (!st.done) atomicAdd(P.active, 1);
  }
}

// ---------------------------------------------------------------------------
// operator-level (parity) kernels
// ---------------------------------------------------------------------------
template <bool WIN>
__global__ void k_eval_mat(DevInst I, DevPop P, int b, int op, MatCands C, const double *lamp, MatDeltas O) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C.n) return;
  Cand c;
  c.r1 = (int)C.r1[i]; c.p1 = (int)C.p1[i]; c.r2 = (int)C.r2[i]; c.p2 = (int)C.p2[i];
  c.l1 = (int)C.len1[i]; c.l2 = (int)C.len2[i]; c.rev1 = C.rev1[i]; c.rev2 = C.rev2[i];
  c.depot = (int)C.depot[i]; c.mode = (int)C.mode[i];
  double lam[4] = {lamp[0], lamp[1], lamp[2], lamp[3]};
  Delta D = eval_cand<WIN>(I, P, b, op, c, lam);
  O.dD[i] = D.dD; O.dV1[i] = D.dV1; O.dV2[i] = D.dV2; O.dV3[i] = D.dV3; O.dV4[i] = D.dV4; O.dF[i] = D.dF;
  O.fn[i] = (unsigned char)D.fn;
}

__global__ void k_emit(DevInst I, DevPop P, int b, int op, long long items, unsigned long long *keys) {
  const int M = P.m[b];
  for (long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (long long)gridDim.x * blockDim.x) {
    Cand c;
    keys[it] = decode_item(I, P, b, op, it, M, c) ? pack_key(c) : 0ull;
  }
}

__global__ void k_totals(DevInst I, DevPop P, int b, double *out) {
  const int m = P.m[b];
  const double4 *RC = P.rcon + (size_t)b * P.J;
  out[0] = pw_sum(RC, 0, m);
  out[1] = pw_sum(RC, 1, m);
  out[2] = pw_sum(RC, 2, m);
  out[3] = pw_sum(RC, 3, m);
  double clo = 0.0;
  for (int r = 0; r < m; r++) clo += (double)P.rmeta[(size_t)b * P.J + r].w;
  out[4] = I.theta * (clo + P.fexcess[b]);
}

__global__ void k_lf_prep(MatCands C, MatDeltas D, unsigned long long *ord, unsigned long long *key,
                          unsigned char *flag, int *nan) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C.n) return;
  Cand c;
  c.r1 = (int)C.r1[i]; c.p1 = (int)C.p1[i]; c.r2 = (int)C.r2[i]; c.p2 = (int)C.p2[i];
  c.l1 = (int)C.len1[i]; c.l2 = (int)C.len2[i]; c.rev1 = C.rev1[i]; c.rev2 = C.rev2[i];
  c.depot = (int)C.depot[i]; c.mode = (int)C.mode[i];
  double f = D.dF[i];
  if (f != f) atomicOr(nan, 1);
  ord[i] = f != f ? ~0ull : ord_of(f);
  key[i] = pack_key(c);
  Delta d;
  d.dD = D.dD[i]; d.dV1 = D.dV1[i]; d.dV2 = D.dV2[i]; d.dV3 = D.dV3[i]; d.dV4 = D.dV4[i]; d.fn = D.fn[i];
  flag[i] = follower_ok(d) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// host <-> device solution transfer (flat layout of mdr_pop_upload)
// ---------------------------------------------------------------------------
__global__ void k_unpack(DevInst I, DevPop P, int B, const int *rbase, const int *coff, const int *cust,
                         const int *dep, const int *arr) {
  int b = blockIdx.x;
  if (b >= B) return;
  int r0 = rbase[b], m = rbase[b + 1] - r0;
  if (threadIdx.x == 0) P.m[b] = m;
  for (int r = threadIdx.x >> 5; r < m; r += blockDim.x >> 5) {
    int c0 = coff[r0 + r], k = coff[r0 + r + 1] - c0;
    int *row = P.seq + row_base(P, b, r);
    for (int p = threadIdx.x & 31; p < k; p += 32) row[p + 1] = cust[c0 + p];
    if ((threadIdx.x & 31) == 0) {
      row[0] = dep[r0 + r];
      if (!I.open) row[k + 1] = arr[r0 + r];
      P.rmeta[(size_t)b * P.J + r] = make_int4(k, dep[r0 + r], arr[r0 + r], 0);
    }
  }
}

// one CTA: flat arrays of all B individuals; hdr = {routes, customers}.  A warp per
// individual counts its routes and customers, two block-wide exclusive scans give every
// individual's route and customer offsets, then a warp per individual writes its rows.
// Shared memory: 2 * B ints (dynamic).
__global__ void __launch_bounds__(1024) k_pack(DevPop P, int b0, int B, int best, int *rbase, int *coff, int *cust,
                                               int *dep, int *arr, int *hdr, int cap_r, int cap_c) {
  extern __shared__ int s_pk[];
  int *s_nr = s_pk, *s_nc = s_pk + B;
  __shared__ int s_tot[2], s_ws[32];
  const int *M = (best ? P.best_m : P.m) + b0;
  const int4 *RM = (best ? P.best_meta : P.rmeta) + (size_t)b0 * P.J;
  const int *SQ = (best ? P.best_seq : P.seq) + (size_t)b0 * P.J * P.Kp;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int b = wid; b < B; b += nw) {
    const int m = M[b];
    int c = 0;
    for (int q = lane; q < m; q += 32) c += RM[(size_t)b * P.J + q].x;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) c += __shfl_xor_sync(0xffffffffu, c, sh);
    if (lane == 0) { s_nr[b] = m; s_nc[b] = c; }
  }
  __syncthreads();
  // exclusive scans of s_nr and s_nc (in place), blockDim-strided chunks with carries
  for (int arrsel = 0; arrsel < 2; arrsel++) {
    int *a = arrsel ? s_nc : s_nr;
    int carry = 0;
    for (int base = 0; base < B; base += blockDim.x) {
      const int i = base + threadIdx.x;
      const int x = i < B ? a[i] : 0;
      int inc = x;
#pragma unroll
      for (int sh = 1; sh < 32; sh <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, sh);
        if (lane >= sh) inc += y;
      }
      if (lane == 31) s_ws[wid] = inc;
      __syncthreads();
      if (wid == 0) {
        int t = lane < nw ? s_ws[lane] : 0;
#pragma unroll
        for (int sh = 1; sh < 32; sh <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, t, sh);
          if (lane >= sh) t += y;
        }
        s_ws[lane] = t;
      }
      __syncthreads();
      const int excl = carry + inc - x + (wid > 0 ? s_ws[wid - 1] : 0);
      const int chunk = s_ws[nw - 1];
      __syncthreads();
      if (i < B) a[i] = excl;
      carry += chunk;
    }
    if (threadIdx.x == 0) s_tot[arrsel] = carry;
    __syncthreads();
  }
  const int R = s_tot[0], Ct = s_tot[1];
  if (threadIdx.x == 0) { hdr[0] = R; hdr[1] = Ct; }
  for (int b = threadIdx.x; b < B; b += blockDim.x) rbase[b] = s_nr[b];
  if (threadIdx.x == 0) rbase[B] = R;
  if (R > cap_r || Ct > cap_c) return;
  for (int b = wid; b < B; b += nw) {
    const int r0 = s_nr[b], m = M[b];
    int c = s_nc[b];
    for (int q = 0; q < m; q++) {
      const int4 mt = RM[(size_t)b * P.J + q];
      const int *row = SQ + ((size_t)b * P.J + q) * P.Kp;
      for (int p = lane; p < mt.x; p += 32) cust[c + p] = row[p + 1];
      if (lane == 0) {
        coff[r0 + q] = c;
        dep[r0 + q] = mt.y;
        arr[r0 + q] = mt.z;
      }
      c += mt.x;
    }
  }
  if (threadIdx.x == 0) coff[R] = Ct;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static size_t select_smem(const DevPop &P) {
  // sel [J] u64, used bitmask, newidx [2J], sm_cnt [ND+4], tl [3J+1] (+ alignment), sorted followers
  return sizeof(unsigned long long) * P.J + sizeof(unsigned) * (P.J / 32 + 1) +
         sizeof(int) * (5 * P.J + P.ND + 8 + 2) + 16 + kSelStageBytes;
}

void launch_rebuild(const DevInst &I, const DevPop &P, int B, bool win, cudaStream_t s) {
  const size_t sm = sizeof(int) * (P.ND + 1) + sizeof(int) * (P.J + 1) + 16 + kRbStageBytes;
  if (sm > 48 * 1024) {  // per device: the attribute call is cheap and launch_rebuild is not in the round graph
    cudaFuncSetAttribute(k_rebuild<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_rebuild<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  }
  if (win) k_rebuild<true><<<B, 256, sm, s>>>(I, P, B);
  else k_rebuild<false><<<B, 256, sm, s>>>(I, P, B);
}

void launch_plan(const DevInst &I, const DevPop &P, const LsParams &L, cudaStream_t s) {
  k_plan<<<1, 1024, 0, s>>>(I, P, L);
}

// launch-configuration caches are per device: attributes set with
// cudaFuncSetAttribute and SM-count grids apply to the device current when set
#define MDR_MAXDEV 16
static int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return (d < 0 || d >= MDR_MAXDEV) ? 0 : d;
}

template <typename K>
static int grid_for(K kern) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0);
  if (per < 1) per = 1;
  return sms * per;
}

int eval_grid_size(bool win) { return win ? grid_for(k_eval<true, 0>) : grid_for(k_eval<false, 0>); }

template <bool WIN>
static void launch_eval_g_region(const DevInst &I, const DevPop &P, const LsParams &L, cudaStream_t s, int region) {
  static int gd[MDR_MAXDEV][3] = {};  // full occupancy of each (latency-bound) form
  int *g = gd[cur_dev()];
  if (!g[0]) {
    g[0] = grid_for(k_eval_g<WIN, -1>);
    g[1] = grid_for(k_eval_g<WIN, 0>);
    g[2] = grid_for(k_eval_g<WIN, 1>);
  }
  // per-producer regions 1 / 2 hold only same-route relocate / swap candidates
  static int generic = -1;  // MDR_G_GENERIC: the generic form for every region (A/B)
  if (generic < 0) generic = getenv("MDR_G_GENERIC") ? 1 : 0;
  const bool spec = P.gbase[1] > 0 && region > 0 && !generic;
  if (spec && region == 1) k_eval_g<WIN, 0><<<g[1], 256, 0, s>>>(I, P, L, region);
  else if (spec) k_eval_g<WIN, 1><<<g[2], 256, 0, s>>>(I, P, L, region);
  else k_eval_g<WIN, -1><<<g[0], 256, 0, s>>>(I, P, L, region);
}

// the three staged evaluators of one (CU, CT) shape on the side streams
// one staged evaluator with its own shape: CU warps per CTA, CT items per task,
// MINB resident CTAs (register budget 64K / (32 CU MINB)), PIPE = the pipelined form
template <bool WIN, int OP, int CU, int CT, int MINB, bool PIPE, int FAM = 0>
static void launch_op(const DevInst &I, const DevPop &P, const LsParams &L, cudaStream_t st) {
  static int gridd[MDR_MAXDEV];
  static size_t smd[MDR_MAXDEV];
  const int dv = cur_dev();
  const size_t smr = sizeof(RBT<WIN>) * (size_t)P.J;
  // 2-opt* (and relocate's warp form) keep per-warp depot-indexed precomputes
  const bool wd = (OP == 2 || (OP == 0 && MDR_REL_WARP)) && I.ND <= MDR_WDMAX;
  const size_t sm = PIPE ? 2 * smr : smr + (wd ? sizeof(double) * 18 * (size_t)I.ND * CU : 0);
  void *fn;
  if constexpr (PIPE) fn = (void *)k_eval_p<WIN, OP, CU, CT, MINB>;
  else fn = (void *)k_eval_c<WIN, OP, CU, CT, MINB, FAM>;
  if (smd[dv] < sm) {
    smd[dv] = sm;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    // shared-memory carveout just large enough for the resident CTAs: the rest of
    // the 228 KB stays L1 for the gathers (+2 % on C4 vs the default)
    cudaFuncAttributes fa;
    size_t stat = 3 * 1024;
    if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess) stat = fa.sharedSizeBytes + 1024;
    int pct = (int)((MINB * (sm + stat) * 100 + 228 * 1024 - 1) / (228 * 1024));
    if (getenv("MDR_CARVEOUT")) pct = atoi(getenv("MDR_CARVEOUT"));
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct);
    cudaFuncSetAttribute(k_eval_g<WIN, -1>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    cudaFuncSetAttribute(k_eval_g<WIN, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    cudaFuncSetAttribute(k_eval_g<WIN, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    gridd[dv] = 0;
  }
  if (!gridd[dv]) {
    int sms = 148, per = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dv);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void *)fn, 32 * CU, sm);
    gridd[dv] = sms * (per < 1 ? 1 : per);
  }
  if constexpr (PIPE) k_eval_p<WIN, OP, CU, CT, MINB><<<gridd[dv], 32 * CU, sm, st>>>(I, P, L);
  else k_eval_c<WIN, OP, CU, CT, MINB, FAM><<<gridd[dv], 32 * CU, sm, st>>>(I, P, L);
}

// swap evaluator shape (large populations): 0 pipelined 16 warps x 128 registers,
// 1 k_eval_c 20 x 96 (default), 2 k_eval_c 24 x 80 (MDR_SWAP_SHAPE overrides)
static int swap_shape(bool win) {
  static int v = -2;
  if (v == -2) v = getenv("MDR_SWAP_SHAPE") ? atoi(getenv("MDR_SWAP_SHAPE")) : -1;
  return v >= 0 ? v : (win ? MDR_SWAP_SHAPE_DEFAULT : 0);  // without windows: pipelined 16 x 128 (C5)
}

// the staged evaluators of a population's shape (only < 0: all three, each on its stream).
// Large shape (>= 100k customers in the population, 32 items per task), per operator,
// measured on C4: relocate 20 warps x 96 registers (k_eval_c), swap 16 x 128 pipelined,
// 2-opt* 24 x 80; small shape: 8 warps x 8 items, 2 CTAs per SM.
template <bool WIN>
static void launch_staged_one(const DevInst &I, const DevPop &P, const LsParams &L, const cudaStream_t *side, int only,
                              bool rel_branch = false) {
  static int pipe_env = -1;
  if (pipe_env < 0) pipe_env = getenv("MDR_NO_PIPE") ? 0 : 1;
  if (P.ct == MDR_LARGE_CT) {
    if (only < 0 || only == 0) {
      // with windows: granular then boundary family as two kernels, each at 24 warps x 80
      // registers (C4 +2.4 %); without windows one kernel at 20 x 96 (the split is -9 % at C5)
      static int split = -1;
      if (split < 0) split = getenv("MDR_REL_SPLIT") ? atoi(getenv("MDR_REL_SPLIT")) : 1;
      if (split && WIN) {
        launch_op<WIN, 0, 8, MDR_LARGE_CT, 3, false, 1>(I, P, L, side[0]);
        // the boundary family on its own branch when the caller gave one (side[3]; joined
        // into side[0] before the intra-route drain), else behind the granular one
        launch_op<WIN, 0, 8, MDR_LARGE_CT, 3, false, 2>(I, P, L, only < 0 && rel_branch ? side[3] : side[0]);
      } else {
        if (MDR_REL_NW_SHAPE == 1) launch_op<WIN, 0, 8, MDR_LARGE_CT, 3, false>(I, P, L, side[0]);
        else launch_op<WIN, 0, 10, MDR_LARGE_CT, 2, false>(I, P, L, side[0]);
      }
    }
    if (only < 0 || only == 1) {
      static int sw_split = -1;
      if (sw_split < 0) sw_split = getenv("MDR_SWAP_SPLIT") ? atoi(getenv("MDR_SWAP_SPLIT")) : 0;
      if (sw_split) {  // v-side segment length 1, then 2: two kernels with half the live state
        launch_op<WIN, 1, 10, MDR_LARGE_CT, 2, false, 1>(I, P, L, side[1]);
        launch_op<WIN, 1, 10, MDR_LARGE_CT, 2, false, 2>(I, P, L, side[1]);
      } else if (swap_shape(WIN) == 1) {
        launch_op<WIN, 1, 10, MDR_LARGE_CT, 2, false>(I, P, L, side[1]);
      } else if (swap_shape(WIN) == 2) {
        launch_op<WIN, 1, 8, MDR_LARGE_CT, 3, false>(I, P, L, side[1]);
      } else if (pipe_env) {
        launch_op<WIN, 1, 16, MDR_LARGE_CT, 1, true>(I, P, L, side[1]);
      } else {
        launch_op<WIN, 1, 16, MDR_LARGE_CT, 1, false>(I, P, L, side[1]);
      }
    }
    if (only < 0 || only == 2) {  // 2-opt*: 24 x 80 with windows (C4 -7 %), 16 x 128 without (C5: 24 warps -24 %)
      if (WIN) launch_op<WIN, 2, 8, MDR_LARGE_CT, MDR_TOS_W_MINB, false>(I, P, L, side[2]);
      else if (MDR_TOS_NW_SHAPE == 1) launch_op<WIN, 2, 8, MDR_LARGE_CT, 3, false>(I, P, L, side[2]);
      else launch_op<WIN, 2, 16, MDR_LARGE_CT, 1, false>(I, P, L, side[2]);
    }
  } else {
    if (only < 0 || only == 0) launch_op<WIN, 0, MDR_SMALL_CU, MDR_SMALL_CT, 2, false>(I, P, L, side[0]);
    if (only < 0 || only == 1) launch_op<WIN, 1, MDR_SMALL_CU, MDR_SMALL_CT, 2, false>(I, P, L, side[1]);
    if (only < 0 || only == 2) launch_op<WIN, 2, MDR_SMALL_CU, MDR_SMALL_CT, 2, false>(I, P, L, side[2]);
  }
}

// kt (profiling only): 7 timing events; the branches are then serialised on s and
// kt[0..6] bracket relocate | its intra drain | swap | its drain | 2-opt* | depot
// enumerators + region-0 drain, so each evaluator's own duration is measured
template <bool WIN>
static void launch_eval_t(const DevInst &I, const DevPop &P, const LsParams &L, cudaStream_t s, const cudaStream_t *side,
                          cudaEvent_t *ev, cudaEvent_t *kt) {
  static int gd[MDR_MAXDEV][6];
  int *g = gd[cur_dev()];
  if (!g[0]) {
    g[0] = grid_for(k_eval<WIN, 0>); g[1] = grid_for(k_eval<WIN, 1>); g[2] = grid_for(k_eval<WIN, 2>);
    g[3] = grid_for(k_eval<WIN, 3>); g[4] = grid_for(k_eval<WIN, 4>); g[5] = grid_for(k_eval<WIN, 5>);
  }
  if (P.staged && kt) {
    const cudaStream_t ser[3] = {s, s, s};
    cudaEventRecord(kt[0], s);
    launch_staged_one<WIN>(I, P, L, ser, 0);
    cudaEventRecord(kt[1], s);
    if (P.gbase[1] > 0) launch_eval_g_region<WIN>(I, P, L, s, 1);
    cudaEventRecord(kt[2], s);
    launch_staged_one<WIN>(I, P, L, ser, 1);
    cudaEventRecord(kt[3], s);
    if (P.gbase[1] > 0) launch_eval_g_region<WIN>(I, P, L, s, 2);
    cudaEventRecord(kt[4], s);
    launch_staged_one<WIN>(I, P, L, ser, 2);
    cudaEventRecord(kt[5], s);
    if (!WIN) k_eval<WIN, 3><<<g[3], 256, 0, s>>>(I, P, L);
    k_eval<WIN, 4><<<g[4], 256, 0, s>>>(I, P, L);
    k_eval<WIN, 5><<<g[5], 256, 0, s>>>(I, P, L);
    if (P.gbase[1] > 0) launch_eval_g_region<WIN>(I, P, L, s, 0);
    cudaEventRecord(kt[6], s);
  } else if (P.staged) {
    // relocate / swap / 2-opt* as parallel branches (fork/join): their
    // persistent grids back-fill each other's tails
    cudaEventRecord(ev[0], s);
    for (int q = 0; q < 4; q++) cudaStreamWaitEvent(side[q], ev[0], 0);
    static int rel_branch = -1;
    if (rel_branch < 0) rel_branch = getenv("MDR_REL_NOBRANCH") ? 0 : 1;
    launch_staged_one<WIN>(I, P, L, side, -1, rel_branch != 0);
    // relocate's boundary family ran on side[3]: join it into side[0] (its drain follows)
    cudaEventRecord(ev[4], side[3]);
    cudaStreamWaitEvent(side[0], ev[4], 0);
    const bool ov0 = P.gbase[1] > 0;
    if (ov0) {  // each producer's intra-route queue drained right behind it, on its branch
      launch_eval_g_region<WIN>(I, P, L, side[0], 1);
      launch_eval_g_region<WIN>(I, P, L, side[1], 2);
    }
    const bool ov = P.gbase[1] > 0;  // per-producer regions (mdr_pop_create; MDR_NO_OVERLAP: single queue)
    if (ov) {  // meanwhile on s: 2-opt / depot enumeration and their generic-path evaluation (region A)
      if (!WIN) k_eval<WIN, 3><<<g[3], 256, 0, s>>>(I, P, L);
      k_eval<WIN, 4><<<g[4], 256, 0, s>>>(I, P, L);
      k_eval<WIN, 5><<<g[5], 256, 0, s>>>(I, P, L);
      launch_eval_g_region<WIN>(I, P, L, s, 0);
    }
    for (int q = 0; q < 3; q++) {
      cudaEventRecord(ev[1 + q], side[q]);
      cudaStreamWaitEvent(s, ev[1 + q], 0);
    }
    if (!ov) {  // the staged evaluators fill the GPU: enumerate after them into the single queue
      if (!WIN) k_eval<WIN, 3><<<g[3], 256, 0, s>>>(I, P, L);
      k_eval<WIN, 4><<<g[4], 256, 0, s>>>(I, P, L);
      k_eval<WIN, 5><<<g[5], 256, 0, s>>>(I, P, L);
    }
  } else {
    k_eval<WIN, 0><<<g[0], 256, 0, s>>>(I, P, L);
    k_eval<WIN, 1><<<g[1], 256, 0, s>>>(I, P, L);
    k_eval<WIN, 2><<<g[2], 256, 0, s>>>(I, P, L);
    if (!WIN) k_eval<WIN, 3><<<g[3], 256, 0, s>>>(I, P, L);
    k_eval<WIN, 4><<<g[4], 256, 0, s>>>(I, P, L);
    k_eval<WIN, 5><<<g[5], 256, 0, s>>>(I, P, L);
  }
}

void launch_eval(const DevInst &I, const DevPop &P, const LsParams &L, int grid, bool win, cudaStream_t s,
                 const cudaStream_t *side, cudaEvent_t *ev, cudaEvent_t *kt) {
  (void)grid;
  if (win) launch_eval_t<true>(I, P, L, s, side, ev, kt);
  else launch_eval_t<false>(I, P, L, s, side, ev, kt);
}

void launch_eval_g(const DevInst &I, const DevPop &P, const LsParams &L, int grid, bool win, cudaStream_t s) {
  (void)grid;  // single-queue mode only: overlap mode drains every region inside launch_eval
  if (P.gbase[1] > 0) return;
  if (win) launch_eval_g_region<true>(I, P, L, s, 1);
  else launch_eval_g_region<false>(I, P, L, s, 1);
}

void launch_select(const DevInst &I, const DevPop &P, const LsParams &L, bool win, cudaStream_t s) {
  size_t sm = select_smem(P);
  static size_t set_td[MDR_MAXDEV], set_fd[MDR_MAXDEV];  // attribute set once per size (not during graph capture)
  const int dv = cur_dev();
  size_t &set_t = set_td[dv], &set_f = set_fd[dv];
  if (win) {
    if (sm > 48 * 1024 && sm > set_t) {
      cudaFuncSetAttribute(k_select<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      set_t = sm;
    }
    k_select<true><<<L.B, MDR_SEL_THREADS, sm, s>>>(I, P, L);
  } else {
    if (sm > 48 * 1024 && sm > set_f) {
      cudaFuncSetAttribute(k_select<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      set_f = sm;
    }
    k_select<false><<<L.B, MDR_SEL_THREADS, sm, s>>>(I, P, L);
  }
}

void launch_eval_mat(const DevInst &I, const DevPop &P, int b, int op, const MatCands &c, const double *lam,
                     MatDeltas out, bool win, cudaStream_t s) {
  if (c.n == 0) return;
  int blocks = (int)((c.n + 255) / 256);
  if (win) k_eval_mat<true><<<blocks, 256, 0, s>>>(I, P, b, op, c, lam, out);
  else k_eval_mat<false><<<blocks, 256, 0, s>>>(I, P, b, op, c, lam, out);
}

void launch_emit(const DevInst &I, const DevPop &P, int b, int op, long long items, unsigned long long *keys,
                 cudaStream_t s) {
  if (items == 0) return;
  long long blocks = (items + 255) / 256;
  if (blocks > 65535) blocks = 65535;
  k_emit<<<(int)blocks, 256, 0, s>>>(I, P, b, op, items, keys);
}

void launch_totals(const DevInst &I, const DevPop &P, int b, double *out, cudaStream_t s) {
  k_totals<<<1, 1, 0, s>>>(I, P, b, out);
}

void launch_unpack(const DevInst &I, const DevPop &P, int B, const int *rbase, const int *coff, const int *cust,
                   const int *dep, const int *arr, cudaStream_t s) {
  k_unpack<<<B, 256, 0, s>>>(I, P, B, rbase, coff, cust, dep, arr);
}

void launch_pack(const DevPop &P, int b0, int B, int best, int *rbase, int *coff, int *cust, int *dep, int *arr,
                 int *hdr, int cap_r, int cap_c, cudaStream_t s) {
  const size_t sm = sizeof(int) * 2 * (size_t)(B > 0 ? B : 1);
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_pack, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_pack<<<1, 1024, sm, s>>>(P, b0, B, best, rbase, coff, cust, dep, arr, hdr, cap_r, cap_c);
}

void launch_lf_prep(const MatCands &c, const MatDeltas &d, unsigned long long *ord, unsigned long long *key,
                    unsigned char *flag, int *nan, cudaStream_t s) {
  if (c.n == 0) return;
  k_lf_prep<<<(int)((c.n + 255) / 256), 256, 0, s>>>(c, d, ord, key, flag, nan);
}

}  // namespace mdr

#ifdef MDR_SEL_PROF
// diagnostic build only (-DMDR_SEL_PROF): k_select phase clocks summed over all CTAs
extern "C" int mdr_debug_selprof(unsigned long long out[16]) {
  return cudaMemcpyFromSymbol(out, mdr::g_selprof, sizeof(unsigned long long) * 16) == cudaSuccess ? 0 : 4;
}
#endif
