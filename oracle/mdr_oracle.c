/*
 * mdr_oracle.c -- scalar CPU restatement of the reference local-search path.
 *
 * TEST INFRASTRUCTURE ONLY (see mdr_oracle.h).  Never on the product path.
 *
 * Exactness rules: compiled with -ffp-contract=off,
 * every numpy expression keeps its left-to-right association, numpy
 * maximum/minimum are a>b?a:b / a<b?a:b, masked (zero-weighted) numpy terms are
 * dropped because they add exact zeros, and an empty subsequence is the exact
 * identity of the concatenation (batch.py:223-262).
 */
#include "mdr_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define EPS 1e-9            /* batch.py:25 */
#define VIOLATION_TOL 1e-9  /* localsearch.py:21 */

enum { RELOCATE = 0, SWAP = 1, TWO_OPT_STAR = 2, TWO_OPT = 3, DEPOT_INSERT = 4, DEPOT_REPLACE = 5 };
enum { MODE_DEPART = 0, MODE_ARRIVE = 1, MODE_BOTH = 2 };

static inline double npmax(double a, double b) { return a > b ? a : b; }
static inline double npmin(double a, double b) { return a < b ? a : b; }

/* ------------------------------------------------------------------------- */
/* subsequence attributes (evaluation.SeqAttr, evaluation.py:22-57)          */
/* ------------------------------------------------------------------------- */
typedef struct {
  double dist, load, T, E, L, TW;
  int first, last;
} attr_t;

static inline attr_t a_empty(void) {
  attr_t a = {0.0, 0.0, 0.0, 0.0, INFINITY, 0.0, -1, -1};
  return a;
}

/* node_attrs / single_attr (batch.py:173-182, evaluation.py:60-71) */
static inline attr_t a_node(const orc_instance_desc *I, int v) {
  attr_t a;
  a.dist = 0.0;
  a.load = I->demand[v];
  a.T = I->service[v];
  a.E = I->has_windows ? I->tw_early[v] : 0.0;
  a.L = I->has_windows ? I->tw_late[v] : INFINITY;
  a.TW = 0.0;
  a.first = a.last = v;
  return a;
}

/* vconcat (batch.py:223-262); empty operands are exact identities */
static inline attr_t a_cat(const orc_instance_desc *I, attr_t a, attr_t b) {
  if (b.first < 0) return a;
  if (a.first < 0) return b;
  size_t lk = (size_t)a.last * (size_t)I->n_nodes + (size_t)b.first;
  double t = I->time[lk];
  double c = I->dist[lk];
  attr_t o;
  o.dist = (a.dist + c) + b.dist;
  o.load = a.load + b.load;
  if (I->has_windows) {
    double delta = (a.T - a.TW) + t;
    double wait = npmax((b.E - delta) - a.L, 0.0);
    double warp = npmax((a.E + delta) - b.L, 0.0);
    o.T = ((a.T + b.T) + t) + wait;
    o.TW = (a.TW + b.TW) + warp;
    o.E = npmax(b.E - delta, a.E) - wait;
    o.L = npmin(b.L - delta, a.L) + warp;
  } else {
    o.T = (a.T + b.T) + t;
    o.E = 0.0;
    o.L = INFINITY;
    o.TW = 0.0;
  }
  o.first = a.first;
  o.last = b.last;
  return o;
}

/* ------------------------------------------------------------------------- */
/* solution + cache                                                          */
/* ------------------------------------------------------------------------- */
typedef struct {
  int dep, arr, k, cap;
  int *c;
} route_t;

typedef struct {
  int m, cap;
  route_t *r;
} sol_t;

typedef struct {
  const orc_instance_desc *I;
  int m;
  int *n, *k, *dep, *arr;
  int64_t *soff, *off2;
  int *seq;
  attr_t *tab; /* full n*n table per route, left fold from i (batch.py:85-124) */
  double *rD, *rV1, *rV2, *rV3, *rclo;
  double *finc, *fdec;
  double fexcess;
  int nv_on;
  /* SolutionIndex (moves.py:151-171) */
  int *route_of, *idx_of, *routed;
  int n_routed;
} cache_t;

static void sol_free(sol_t *s) {
  for (int i = 0; i < s->cap; i++) free(s->r[i].c);
  free(s->r);
  s->r = NULL;
  s->m = s->cap = 0;
}

static void route_set(route_t *r, int dep, int arr, const int *c, int k) {
  if (r->cap < k) {
    int nc = k < 8 ? 8 : k * 2;
    r->c = (int *)realloc(r->c, sizeof(int) * (size_t)nc);
    r->cap = nc;
  }
  if (k) memmove(r->c, c, sizeof(int) * (size_t)k);
  r->k = k;
  r->dep = dep;
  r->arr = arr;
}

static void sol_reserve(sol_t *s, int m) {
  if (s->cap >= m) return;
  int nc = m < 16 ? 16 : m * 2;
  s->r = (route_t *)realloc(s->r, sizeof(route_t) * (size_t)nc);
  memset(s->r + s->cap, 0, sizeof(route_t) * (size_t)(nc - s->cap));
  s->cap = nc;
}

static void sol_from_flat(sol_t *s, const orc_flat_sol *f) {
  memset(s, 0, sizeof(*s));
  sol_reserve(s, f->m);
  s->m = f->m;
  for (int r = 0; r < f->m; r++)
    route_set(&s->r[r], f->depart[r], f->arrive[r], f->cust + f->off[r], f->off[r + 1] - f->off[r]);
}

/* _route_penalties (batch.py:271-293) for one route; zeros when empty */
static inline void contrib(const orc_instance_desc *I, const attr_t *a, int dep, int arr,
                           int64_t kcount, double out[5]) {
  if (kcount <= 0) {
    out[0] = out[1] = out[2] = out[3] = out[4] = 0.0;
    return;
  }
  out[0] = a->dist;
  out[1] = I->has_windows ? I->gamma * a->TW : 0.0;
  out[2] = (I->theta * npmax(a->load - I->capacity, 0.0)) / I->capacity;
  out[3] = isinf(I->max_duration) ? 0.0
                                  : (I->theta * npmax(a->T - I->max_duration, 0.0)) / I->max_duration;
  out[4] = I->open_routes ? 0.0 : (dep != arr ? 1.0 : 0.0);
}

static void cache_free(cache_t *C) {
  free(C->n); free(C->k); free(C->dep); free(C->arr); free(C->soff); free(C->off2);
  free(C->seq); free(C->tab); free(C->rD); free(C->rV1); free(C->rV2); free(C->rV3);
  free(C->rclo); free(C->finc); free(C->fdec); free(C->route_of); free(C->idx_of);
  free(C->routed);
  memset(C, 0, sizeof(*C));
}

static void cache_build(cache_t *C, const orc_instance_desc *I, const sol_t *s) {
  memset(C, 0, sizeof(*C));
  C->I = I;
  int m = s->m;
  C->m = m;
  C->n = (int *)calloc((size_t)m + 1, sizeof(int));
  C->k = (int *)calloc((size_t)m + 1, sizeof(int));
  C->dep = (int *)calloc((size_t)m + 1, sizeof(int));
  C->arr = (int *)calloc((size_t)m + 1, sizeof(int));
  C->soff = (int64_t *)calloc((size_t)m + 1, sizeof(int64_t));
  C->off2 = (int64_t *)calloc((size_t)m + 1, sizeof(int64_t));
  for (int r = 0; r < m; r++) {
    C->k[r] = s->r[r].k;
    C->dep[r] = s->r[r].dep;
    C->arr[r] = s->r[r].arr;
    C->n[r] = s->r[r].k + (I->open_routes ? 1 : 2); /* Route.sequence model.py:168-171 */
    C->soff[r + 1] = C->soff[r] + C->n[r];
    C->off2[r + 1] = C->off2[r] + (int64_t)C->n[r] * C->n[r];
  }
  C->seq = (int *)malloc(sizeof(int) * (size_t)(C->soff[m] + 1));
  for (int r = 0; r < m; r++) {
    int *q = C->seq + C->soff[r];
    q[0] = s->r[r].dep;
    for (int i = 0; i < s->r[r].k; i++) q[i + 1] = s->r[r].c[i];
    if (!I->open_routes) q[s->r[r].k + 1] = s->r[r].arr;
  }
  /* tables: entry (r,i,j) = left fold from i of positions i..j (batch.py:85-124).
   * Entries with j<i keep the zero/inf initialisation of batch.py:75-81. */
  C->tab = (attr_t *)malloc(sizeof(attr_t) * (size_t)(C->off2[m] + 1));
  for (int64_t e = 0; e < C->off2[m] + 1; e++) {
    C->tab[e] = a_empty();
    C->tab[e].first = C->tab[e].last = 0;
  }
  for (int r = 0; r < m; r++) {
    int n = C->n[r];
    const int *q = C->seq + C->soff[r];
    for (int i = 0; i < n; i++) {
      attr_t acc = a_node(I, q[i]);
      C->tab[C->off2[r] + (int64_t)i * n + i] = acc;
      for (int j = i + 1; j < n; j++) {
        acc = a_cat(I, acc, a_node(I, q[j]));
        C->tab[C->off2[r] + (int64_t)i * n + j] = acc;
      }
    }
  }
  /* per-route contributions (batch.py:126-142) */
  C->rD = (double *)calloc((size_t)m + 1, sizeof(double));
  C->rV1 = (double *)calloc((size_t)m + 1, sizeof(double));
  C->rV2 = (double *)calloc((size_t)m + 1, sizeof(double));
  C->rV3 = (double *)calloc((size_t)m + 1, sizeof(double));
  C->rclo = (double *)calloc((size_t)m + 1, sizeof(double));
  for (int r = 0; r < m; r++) {
    attr_t full = C->tab[C->off2[r] + (C->n[r] - 1)];
    double o[5];
    contrib(I, &full, C->dep[r], C->arr[r], C->k[r], o);
    /* route_D is the raw table distance even for empty routes (batch.py:129) */
    C->rD[r] = full.dist;
    C->rV1[r] = o[1];
    C->rV2[r] = o[2];
    C->rV3[r] = o[3];
    C->rclo[r] = o[4];
  }
  /* depot counts and fleet increments (batch.py:144-158) */
  int nd = I->n_depots;
  C->finc = (double *)calloc((size_t)nd, sizeof(double));
  C->fdec = (double *)calloc((size_t)nd, sizeof(double));
  C->nv_on = !isinf(I->fleet_per_depot);
  C->fexcess = 0.0;
  if (C->nv_on) {
    int64_t *cnt = (int64_t *)calloc((size_t)nd, sizeof(int64_t));
    for (int r = 0; r < m; r++)
      if (C->k[r] > 0) cnt[C->dep[r]]++;
    double nv = I->fleet_per_depot;
    for (int d = 0; d < nd; d++) {
      double c = (double)cnt[d];
      double over = npmax(c - nv, 0.0);
      C->finc[d] = npmax((c + 1.0) - nv, 0.0) - over;
      C->fdec[d] = npmax((c - 1.0) - nv, 0.0) - over;
      C->fexcess += over;
    }
    free(cnt);
  }
  /* SolutionIndex */
  int N = I->n_nodes;
  C->route_of = (int *)malloc(sizeof(int) * (size_t)N);
  C->idx_of = (int *)malloc(sizeof(int) * (size_t)N);
  for (int v = 0; v < N; v++) C->route_of[v] = C->idx_of[v] = -1;
  for (int r = 0; r < m; r++)
    for (int i = 0; i < s->r[r].k; i++) {
      C->route_of[s->r[r].c[i]] = r;
      C->idx_of[s->r[r].c[i]] = i;
    }
  C->routed = (int *)malloc(sizeof(int) * (size_t)(N + 1));
  C->n_routed = 0;
  for (int v = I->n_depots; v < N; v++)
    if (C->route_of[v] >= 0) C->routed[C->n_routed++] = v;
}

/* SolutionCache.gather (batch.py:184-221) for one candidate */
static inline attr_t gather(const cache_t *C, int r, int64_t i, int64_t j, int allow_empty, int swap) {
  if (j < i) {
    if (allow_empty) return a_empty();
    /* out-of-contract read of the reference (only reachable for k=0 routes,
     * whose contributions are masked); return a harmless non-empty value */
    attr_t z = a_empty();
    z.first = z.last = C->seq[C->soff[r]];
    return z;
  }
  int n = C->n[r];
  attr_t a = C->tab[C->off2[r] + i * n + j];
  a.first = C->seq[C->soff[r] + i];
  a.last = C->seq[C->soff[r] + j];
  if (swap) {
    int t = a.first;
    a.first = a.last;
    a.last = t;
  }
  return a;
}

typedef struct {
  int64_t r1, p1, r2, p2, len1, len2, depot, mode;
  int rev1, rev2;
} cand_t;

/* evaluate_candidates (batch.py:365-553) for one candidate */
static void eval_one(const cache_t *C, int op, const cand_t *c, const double lam[4], double out[6],
                     uint8_t *fneutral) {
  const orc_instance_desc *I = C->I;
  double nw[5] = {0, 0, 0, 0, 0}, old[5], cA[5], cB[5];
  double fleet_delta = 0.0;
  int fn = 1;
  int r1 = (int)c->r1, r2 = (int)c->r2;
  int64_t p1 = c->p1, p2 = c->p2, l1 = c->len1, l2 = c->len2;
  int n1 = C->n[r1];
  int two_routes = 0;

  switch (op) {
  case RELOCATE: {
    attr_t seg = gather(C, r1, p1 + 1, p1 + l1, 0, c->rev1);
    if (r1 == r2) {
      int before = p2 <= p1;
      attr_t pref = gather(C, r1, 0, before ? p2 : p1, 0, 0);
      attr_t mid = before ? gather(C, r1, p2 + 1, p1, 1, 0) : gather(C, r1, p1 + l1 + 1, p2, 1, 0);
      attr_t suf = gather(C, r1, before ? p1 + l1 + 1 : p2 + 1, n1 - 1, 1, 0);
      attr_t x = before ? a_cat(I, a_cat(I, pref, seg), mid) : a_cat(I, a_cat(I, pref, mid), seg);
      x = a_cat(I, x, suf);
      contrib(I, &x, C->dep[r1], C->arr[r1], C->k[r1], cA);
      for (int f = 0; f < 5; f++) nw[f] = 0.0 + cA[f];
    } else {
      two_routes = 1;
      int n2 = C->n[r2];
      attr_t newA = a_cat(I, gather(C, r1, 0, p1, 0, 0), gather(C, r1, p1 + l1 + 1, n1 - 1, 1, 0));
      attr_t newB = a_cat(I, a_cat(I, gather(C, r2, 0, p2, 0, 0), seg), gather(C, r2, p2 + 1, n2 - 1, 1, 0));
      int64_t kA = C->k[r1] - l1, kB = C->k[r2] + l1;
      contrib(I, &newA, C->dep[r1], C->arr[r1], kA, cA);
      contrib(I, &newB, C->dep[r2], C->arr[r2], kB, cB);
      for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
      if (C->nv_on && kA == 0) {
        fleet_delta = 0.0 + C->fdec[C->dep[r1]];
        fn = 0;
      }
    }
    break;
  }
  case SWAP: {
    attr_t segA = gather(C, r1, p1 + 1, p1 + l1, 0, c->rev1);
    if (r1 == r2) {
      attr_t segB = gather(C, r1, p2 + 1, p2 + l2, 1, c->rev2);
      attr_t x = a_cat(I, gather(C, r1, 0, p1, 0, 0), segB);
      x = a_cat(I, x, gather(C, r1, p1 + l1 + 1, p2, 1, 0));
      x = a_cat(I, x, segA);
      x = a_cat(I, x, gather(C, r1, p2 + l2 + 1, n1 - 1, 1, 0));
      contrib(I, &x, C->dep[r1], C->arr[r1], C->k[r1], cA);
      for (int f = 0; f < 5; f++) nw[f] = 0.0 + cA[f];
    } else {
      two_routes = 1;
      int n2 = C->n[r2];
      attr_t segB = gather(C, r2, p2 + 1, p2 + l2, 1, c->rev2);
      attr_t newA = a_cat(I, a_cat(I, gather(C, r1, 0, p1, 0, 0), segB),
                          gather(C, r1, p1 + l1 + 1, n1 - 1, 1, 0));
      attr_t newB = a_cat(I, a_cat(I, gather(C, r2, 0, p2, 0, 0), segA),
                          gather(C, r2, p2 + l2 + 1, n2 - 1, 1, 0));
      int64_t kA = C->k[r1] - l1 + l2, kB = C->k[r2] - l2 + l1;
      contrib(I, &newA, C->dep[r1], C->arr[r1], kA, cA);
      contrib(I, &newB, C->dep[r2], C->arr[r2], kB, cB);
      for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
    }
    break;
  }
  case TWO_OPT: {
    attr_t x = a_cat(I, gather(C, r1, 0, p1, 0, 0), gather(C, r1, p1 + 1, p2 + 1, 0, 1));
    x = a_cat(I, x, gather(C, r1, p2 + 2, n1 - 1, 1, 0));
    contrib(I, &x, C->dep[r1], C->arr[r1], C->k[r1], cA);
    for (int f = 0; f < 5; f++) nw[f] = 0.0 + cA[f];
    break;
  }
  case TWO_OPT_STAR: {
    two_routes = 1;
    int n2 = C->n[r2];
    attr_t newA = a_cat(I, gather(C, r1, 0, p1, 0, 0), gather(C, r2, p2 + 1, n2 - 1, 1, 0));
    attr_t newB = a_cat(I, gather(C, r2, 0, p2, 0, 0), gather(C, r1, p1 + 1, n1 - 1, 1, 0));
    int64_t kA = p1 + (C->k[r2] - p2), kB = p2 + (C->k[r1] - p1);
    contrib(I, &newA, C->dep[r1], C->arr[r2], kA, cA);
    contrib(I, &newB, C->dep[r2], C->arr[r1], kB, cB);
    for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
    if (C->nv_on) {
      fleet_delta = (0.0 + (kA == 0 ? C->fdec[C->dep[r1]] : 0.0)) + (kB == 0 ? C->fdec[C->dep[r2]] : 0.0);
      fn = (kA > 0) && (kB > 0);
    }
    break;
  }
  case DEPOT_INSERT: {
    int d = (int)c->depot;
    int64_t k1 = C->k[r1];
    attr_t head = gather(C, r1, 0, p1, 0, 0), tail;
    if (!I->open_routes) {
      head = a_cat(I, head, a_node(I, C->arr[r1]));
      tail = a_cat(I, a_cat(I, a_node(I, d), gather(C, r1, p1 + 1, k1, 0, 0)), a_node(I, d));
    } else {
      tail = a_cat(I, a_node(I, d), gather(C, r1, p1 + 1, k1, 0, 0));
    }
    contrib(I, &head, C->dep[r1], C->arr[r1], p1, cA);
    contrib(I, &tail, d, d, k1 - p1, cB);
    for (int f = 0; f < 5; f++) nw[f] = (0.0 + cA[f]) + cB[f];
    if (C->nv_on) {
      int drops = p1 == 0, same_dep = d == C->dep[r1];
      double fd = (drops && same_dep) ? 0.0 : (drops ? C->finc[d] + C->fdec[C->dep[r1]] : C->finc[d]);
      fleet_delta = 0.0 + fd;
      fn = 0;
    }
    break;
  }
  case DEPOT_REPLACE: {
    int d = (int)c->depot, mode = (int)c->mode;
    int dep_new = mode != MODE_ARRIVE ? d : C->dep[r1];
    int arr_new = mode != MODE_DEPART ? d : C->arr[r1];
    attr_t x0 = mode == MODE_ARRIVE ? a_empty() : a_node(I, dep_new);
    int64_t i0 = mode == MODE_ARRIVE ? 0 : 1;
    attr_t x;
    if (I->open_routes) {
      x = a_cat(I, x0, gather(C, r1, i0, n1 - 1, 0, 0));
    } else {
      int64_t j0 = mode == MODE_DEPART ? n1 - 1 : n1 - 2;
      attr_t x2 = mode == MODE_DEPART ? a_empty() : a_node(I, arr_new);
      x = a_cat(I, a_cat(I, x0, gather(C, r1, i0, j0, 0, 0)), x2);
    }
    contrib(I, &x, dep_new, arr_new, C->k[r1], cA);
    for (int f = 0; f < 5; f++) nw[f] = 0.0 + cA[f];
    if (C->nv_on) {
      int moves_dep = dep_new != C->dep[r1];
      if (moves_dep) fleet_delta = 0.0 + (C->finc[dep_new] + C->fdec[C->dep[r1]]);
      fn = !moves_dep;
    }
    break;
  }
  default:
    for (int f = 0; f < 6; f++) out[f] = NAN;
    *fneutral = 0;
    return;
  }
  /* _old_contrib (batch.py:342-357) */
  old[0] = C->rD[r1]; old[1] = C->rV1[r1]; old[2] = C->rV2[r1]; old[3] = C->rV3[r1]; old[4] = C->rclo[r1];
  if (two_routes) {
    old[0] = old[0] + C->rD[r2];
    old[1] = old[1] + C->rV1[r2];
    old[2] = old[2] + C->rV2[r2];
    old[3] = old[3] + C->rV3[r2];
    old[4] = old[4] + C->rclo[r2];
  }
  /* combine (batch.py:545-553) */
  double dD = nw[0] - old[0];
  double dV1 = nw[1] - old[1];
  double dV2 = nw[2] - old[2];
  double dV3 = nw[3] - old[3];
  double dV4 = I->theta * ((nw[4] - old[4]) + fleet_delta);
  out[0] = dD; out[1] = dV1; out[2] = dV2; out[3] = dV3; out[4] = dV4;
  out[5] = (((dD + lam[0] * dV1) + lam[1] * dV2) + lam[2] * dV3) + lam[3] * dV4;
  *fneutral = (uint8_t)fn;
}

/* ------------------------------------------------------------------------- */
/* enumeration (moves.py:253-464), reference order                           */
/* ------------------------------------------------------------------------- */
typedef struct {
  orc_cands *cs;
  int64_t cap, n;
  int overflow;
} emit_t;

static inline void emit(emit_t *E, int64_t r1, int64_t p1, int64_t r2, int64_t p2, int64_t l1, int64_t l2,
                        int b1, int b2, int64_t depot, int64_t mode) {
  if (E->cs) {
    if (E->n >= E->cap) {
      E->overflow = 1;
    } else {
      orc_cands *c = E->cs;
      int64_t i = E->n;
      c->r1[i] = r1; c->p1[i] = p1; c->r2[i] = r2; c->p2[i] = p2; c->len1[i] = l1; c->len2[i] = l2;
      c->rev1[i] = (uint8_t)b1; c->rev2[i] = (uint8_t)b2; c->depot[i] = depot; c->mode[i] = mode;
    }
  }
  E->n++;
}

/* iterate _neighbor_pairs (moves.py:253-268): u ascending, list slot order */
#define FOR_PAIRS(C, u, v)                                                                         \
  for (int u = (C)->I->n_depots; u < (C)->I->n_nodes; u++)                                         \
    for (int _s = 0, v; _s < (C)->I->width; _s++)                                                  \
      if ((v = (C)->I->lists[(size_t)u * (C)->I->width + _s]) >= 0 && (C)->route_of[u] >= 0 &&     \
          (C)->route_of[v] >= 0)

static void enum_op(const cache_t *C, int op, emit_t *E) {
  const orc_instance_desc *I = C->I;
  int symmetric = !I->has_windows;
  int M = C->m;
  if (op == RELOCATE) { /* moves.py:280-311 */
    int nvar = symmetric ? 3 : 2;
    static const int VL[3] = {1, 2, 2}, VR[3] = {0, 0, 1};
    for (int vi = 0; vi < nvar; vi++) {
      int len = VL[vi], rev = VR[vi];
      FOR_PAIRS(C, u, v) {
        int ru = C->route_of[u], pu = C->idx_of[u], rv = C->route_of[v], pv = C->idx_of[v];
        int ku = C->k[ru], same = ru == rv, tgt = pv + 1;
        int fits = pu + len <= ku;
        int inside = same && tgt > pu && tgt <= pu + len;
        int ok = fits && !inside && !(same && tgt == pu + len);
        if (!rev) ok = ok && !(same && tgt == pu);
        if (ok) emit(E, ru, pu, rv, tgt, len, 0, rev, 0, -1, -1);
      }
      for (int front = 1; front >= 0; front--)
        for (int a = 0; a < C->n_routed; a++) {
          int ub = C->routed[a], rub = C->route_of[ub], pub = C->idx_of[ub], kub = C->k[rub];
          for (int rb = 0; rb < M; rb++) {
            int tg = front ? 0 : C->k[rb], sameb = rub == rb;
            int ok = (pub + len <= kub) && !(sameb && tg == pub + len);
            if (!rev) ok = ok && !(sameb && tg == pub);
            if (ok) emit(E, rub, pub, rb, tg, len, 0, rev, 0, -1, -1);
          }
        }
    }
  } else if (op == SWAP) { /* moves.py:314-358 */
    int combos[9][4], nc = 0;
    if (symmetric) {
      for (int lu = 1; lu <= 2; lu++)
        for (int lv = 1; lv <= 2; lv++)
          for (int au = 0; au <= (lu == 2); au++)
            for (int av = 0; av <= (lv == 2); av++) {
              combos[nc][0] = lu; combos[nc][1] = lv; combos[nc][2] = au; combos[nc][3] = av; nc++;
            }
    } else {
      static const int base[4][2] = {{1, 1}, {1, 2}, {2, 1}, {2, 2}};
      for (int i = 0; i < 4; i++) {
        combos[nc][0] = base[i][0]; combos[nc][1] = base[i][1]; combos[nc][2] = 0; combos[nc][3] = 0; nc++;
      }
    }
    for (int ci = 0; ci < nc; ci++) {
      int lu = combos[ci][0], lv = combos[ci][1], au = combos[ci][2], av = combos[ci][3];
      FOR_PAIRS(C, u, v) {
        if (u == v) continue;
        int ru = C->route_of[u], pu = C->idx_of[u], rv = C->route_of[v], pv = C->idx_of[v];
        int same = ru == rv, flip = same && pu > pv;
        int q1 = flip ? pv : pu, q2 = flip ? pu : pv;
        int l1 = flip ? lv : lu, l2 = flip ? lu : lv;
        int b1 = flip ? av : au, b2 = flip ? au : av;
        int fits = (q1 + l1 <= C->k[ru]) && (q2 + l2 <= C->k[rv]);
        if (fits && (!same || q2 >= q1 + l1)) emit(E, ru, q1, rv, q2, l1, l2, b1, b2, -1, -1);
      }
    }
  } else if (op == TWO_OPT) { /* moves.py:361-372 */
    if (I->has_windows) return;
    for (int dir = 0; dir < 2; dir++) {
      FOR_PAIRS(C, u, v) {
        int ru = C->route_of[u], pu = C->idx_of[u], rv = C->route_of[v], pv = C->idx_of[v];
        if (ru != rv) continue;
        if (dir == 0 && pv >= pu + 2) emit(E, ru, pu + 1, -1, pv, 0, 0, 0, 0, -1, -1);
        if (dir == 1 && pu >= pv + 2) emit(E, ru, pv + 1, -1, pu, 0, 0, 0, 0, -1, -1);
      }
    }
  } else if (op == TWO_OPT_STAR) { /* moves.py:375-405 */
    if (M < 2) return;
    FOR_PAIRS(C, u, v) {
      int ru = C->route_of[u], rv = C->route_of[v];
      if (ru != rv) emit(E, ru, C->idx_of[u] + 1, rv, C->idx_of[v], 0, 0, 0, 0, -1, -1);
    }
    for (int a = 0; a < C->n_routed; a++) {
      int ub = C->routed[a], rub = C->route_of[ub], pub = C->idx_of[ub];
      for (int rb = 0; rb < M; rb++) {
        if (rub == rb) continue;
        int q1 = pub + 1, q2 = C->k[rb];
        int dropb = (q1 == C->k[rub]) && (q2 == C->k[rb]);
        if (!I->open_routes) dropb = dropb && (C->arr[rub] == C->arr[rb]);
        if (!dropb) emit(E, rub, q1, rb, q2, 0, 0, 0, 0, -1, -1);
      }
    }
    for (int a = 0; a < C->n_routed; a++) {
      int ub = C->routed[a], rub = C->route_of[ub], pub = C->idx_of[ub];
      for (int rb = 0; rb < M; rb++)
        if (rub != rb) emit(E, rb, 0, rub, pub, 0, 0, 0, 0, -1, -1);
    }
    for (int ra = 0; ra < M; ra++)
      for (int rb = 0; rb < M; rb++)
        if (ra != rb) emit(E, ra, 0, rb, C->k[rb], 0, 0, 0, 0, -1, -1);
  } else if (op == DEPOT_INSERT) { /* moves.py:408-422 */
    for (int r = 0; r < M; r++) {
      if (C->k[r] <= 0) continue;
      int closes_same = I->open_routes || C->arr[r] == C->dep[r];
      for (int p = 0; p < C->k[r]; p++)
        for (int d = 0; d < I->n_depots; d++) {
          if (p == 0 && d == C->dep[r] && closes_same) continue;
          emit(E, r, p, -1, -1, 0, 0, 0, 0, d, -1);
        }
    }
  } else if (op == DEPOT_REPLACE) { /* moves.py:425-441 */
    int nmodes = I->open_routes ? 1 : 3;
    for (int mode = 0; mode < nmodes; mode++)
      for (int r = 0; r < M; r++)
        for (int d = 0; d < I->n_depots; d++) {
          int ok;
          if (mode == MODE_DEPART) ok = d != C->dep[r];
          else if (mode == MODE_ARRIVE) ok = d != C->arr[r];
          else ok = !(d == C->dep[r] && d == C->arr[r]);
          if (ok) emit(E, r, 0, -1, -1, 0, 0, 0, 0, d, mode);
        }
  }
}

/* ------------------------------------------------------------------------- */
/* leader / followers (batch.py:578-614)                                     */
/* ------------------------------------------------------------------------- */
static inline int key_cmp(const orc_cands *cs, int64_t a, int64_t b) {
  /* moves.key_arrays (moves.py:210-213): r1, r2, p1, p2, len1, len2, rev1, rev2, depot, mode */
#define KC(F) if (cs->F[a] != cs->F[b]) return cs->F[a] < cs->F[b] ? -1 : 1;
  KC(r1) KC(r2) KC(p1) KC(p2) KC(len1) KC(len2) KC(rev1) KC(rev2) KC(depot) KC(mode)
#undef KC
  return 0;
}

typedef struct {
  const orc_cands *cs;
  const double *dF;
} sort_ctx_t;


static int fol_less(const sort_ctx_t *S, int64_t a, int64_t b) {
  /* np.lexsort(keys + (dF,)) -- dF primary (numeric, -0 == +0), key, then index (stable) */
  double fa = S->dF[a], fb = S->dF[b];
  if (fa < fb) return 1;
  if (fa > fb) return 0;
  int kc = key_cmp(S->cs, a, b);
  if (kc) return kc < 0;
  return a < b;
}

static void msort(const sort_ctx_t *S, int64_t *v, int64_t *tmp, int64_t n) {
  if (n < 2) return;
  int64_t h = n / 2;
  msort(S, v, tmp, h);
  msort(S, v + h, tmp, n - h);
  int64_t i = 0, j = h, o = 0;
  while (i < h && j < n) tmp[o++] = fol_less(S, v[j], v[i]) ? v[j++] : v[i++];
  while (i < h) tmp[o++] = v[i++];
  while (j < n) tmp[o++] = v[j++];
  memcpy(v, tmp, sizeof(int64_t) * (size_t)n);
}

int64_t orc_leader_followers(const orc_cands *cs, const orc_deltas *d, int32_t multi_move,
                             int64_t *followers, int64_t *n_followers) {
  int64_t n = cs->n;
  if (n_followers) *n_followers = 0;
  if (n == 0) return -1;
  double best_val = d->dF[0];
  for (int64_t i = 0; i < n; i++) {
    if (isnan(d->dF[i])) return -1; /* numpy min propagates NaN */
    if (d->dF[i] < best_val) best_val = d->dF[i];
  }
  if (!(best_val < -EPS)) return -1;
  int64_t best = -1;
  for (int64_t i = 0; i < n; i++)
    if (d->dF[i] == best_val && (best < 0 || key_cmp(cs, i, best) < 0)) best = i;
  if (multi_move && followers) {
    int64_t nf = 0;
    for (int64_t i = 0; i < n; i++) {
      if (i == best) continue;
      if (d->dD[i] < -EPS && fabs(d->dV1[i]) <= EPS && fabs(d->dV2[i]) <= EPS &&
          fabs(d->dV3[i]) <= EPS && fabs(d->dV4[i]) <= EPS && d->fleet_neutral[i])
        followers[nf++] = i;
    }
    sort_ctx_t S = {cs, d->dF};
    int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nf + 1));
    msort(&S, followers, tmp, nf);
    free(tmp);
    *n_followers = nf;
  }
  return best;
}

/* ------------------------------------------------------------------------- */
/* apply (moves.move_plan moves.py:88-148, localsearch.apply_moves :58-82)   */
/* ------------------------------------------------------------------------- */
typedef struct {
  int idx; /* -1 = new route */
  int dep, arr, k;
  int *c;
} plan_t;

static int plan_move(const sol_t *s, int op, const cand_t *mv, plan_t out[2]) {
  const route_t *ra = &s->r[mv->r1];
  int p1 = (int)mv->p1, p2 = (int)mv->p2, l1 = (int)mv->len1, l2 = (int)mv->len2;
  switch (op) {
  case RELOCATE: {
    int seg[2];
    for (int i = 0; i < l1; i++) seg[i] = ra->c[p1 + i];
    if (mv->rev1 && l1 == 2) { int t = seg[0]; seg[0] = seg[1]; seg[1] = t; }
    if (mv->r1 == mv->r2) {
      int *rest = (int *)malloc(sizeof(int) * (size_t)(ra->k + 1)), nr = 0;
      for (int i = 0; i < ra->k; i++)
        if (i < p1 || i >= p1 + l1) rest[nr++] = ra->c[i];
      int at = p2 > p1 ? p2 - l1 : p2;
      int *c = (int *)malloc(sizeof(int) * (size_t)(ra->k + 1)), k = 0;
      for (int i = 0; i < at; i++) c[k++] = rest[i];
      for (int i = 0; i < l1; i++) c[k++] = seg[i];
      for (int i = at; i < nr; i++) c[k++] = rest[i];
      free(rest);
      out[0] = (plan_t){(int)mv->r1, ra->dep, ra->arr, k, c};
      return 1;
    }
    const route_t *rb = &s->r[mv->r2];
    int *ca = (int *)malloc(sizeof(int) * (size_t)(ra->k + 1)), ka = 0;
    for (int i = 0; i < ra->k; i++)
      if (i < p1 || i >= p1 + l1) ca[ka++] = ra->c[i];
    int *cb = (int *)malloc(sizeof(int) * (size_t)(rb->k + l1 + 1)), kb = 0;
    for (int i = 0; i < p2; i++) cb[kb++] = rb->c[i];
    for (int i = 0; i < l1; i++) cb[kb++] = seg[i];
    for (int i = p2; i < rb->k; i++) cb[kb++] = rb->c[i];
    out[0] = (plan_t){(int)mv->r1, ra->dep, ra->arr, ka, ca};
    out[1] = (plan_t){(int)mv->r2, rb->dep, rb->arr, kb, cb};
    return 2;
  }
  case SWAP: {
    int s1[2], s2[2];
    for (int i = 0; i < l1; i++) s1[i] = ra->c[p1 + i];
    if (mv->rev1 && l1 == 2) { int t = s1[0]; s1[0] = s1[1]; s1[1] = t; }
    const route_t *rb = mv->r1 == mv->r2 ? ra : &s->r[mv->r2];
    for (int i = 0; i < l2; i++) s2[i] = rb->c[p2 + i];
    if (mv->rev2 && l2 == 2) { int t = s2[0]; s2[0] = s2[1]; s2[1] = t; }
    if (mv->r1 == mv->r2) {
      int *c = (int *)malloc(sizeof(int) * (size_t)(ra->k + 4)), k = 0;
      for (int i = 0; i < p1; i++) c[k++] = ra->c[i];
      for (int i = 0; i < l2; i++) c[k++] = s2[i];
      for (int i = p1 + l1; i < p2; i++) c[k++] = ra->c[i];
      for (int i = 0; i < l1; i++) c[k++] = s1[i];
      for (int i = p2 + l2; i < ra->k; i++) c[k++] = ra->c[i];
      out[0] = (plan_t){(int)mv->r1, ra->dep, ra->arr, k, c};
      return 1;
    }
    int *ca = (int *)malloc(sizeof(int) * (size_t)(ra->k + 4)), ka = 0;
    for (int i = 0; i < p1; i++) ca[ka++] = ra->c[i];
    for (int i = 0; i < l2; i++) ca[ka++] = s2[i];
    for (int i = p1 + l1; i < ra->k; i++) ca[ka++] = ra->c[i];
    int *cb = (int *)malloc(sizeof(int) * (size_t)(rb->k + 4)), kb = 0;
    for (int i = 0; i < p2; i++) cb[kb++] = rb->c[i];
    for (int i = 0; i < l1; i++) cb[kb++] = s1[i];
    for (int i = p2 + l2; i < rb->k; i++) cb[kb++] = rb->c[i];
    out[0] = (plan_t){(int)mv->r1, ra->dep, ra->arr, ka, ca};
    out[1] = (plan_t){(int)mv->r2, rb->dep, rb->arr, kb, cb};
    return 2;
  }
  case TWO_OPT: {
    int *c = (int *)malloc(sizeof(int) * (size_t)(ra->k + 1)), k = 0;
    for (int i = 0; i < p1; i++) c[k++] = ra->c[i];
    for (int i = p2; i >= p1; i--) c[k++] = ra->c[i];
    for (int i = p2 + 1; i < ra->k; i++) c[k++] = ra->c[i];
    out[0] = (plan_t){(int)mv->r1, ra->dep, ra->arr, k, c};
    return 1;
  }
  case TWO_OPT_STAR: {
    const route_t *rb = &s->r[mv->r2];
    int *ca = (int *)malloc(sizeof(int) * (size_t)(ra->k + rb->k + 1)), ka = 0;
    int *cb = (int *)malloc(sizeof(int) * (size_t)(ra->k + rb->k + 1)), kb = 0;
    for (int i = 0; i < p1; i++) ca[ka++] = ra->c[i];
    for (int i = p2; i < rb->k; i++) ca[ka++] = rb->c[i];
    for (int i = 0; i < p2; i++) cb[kb++] = rb->c[i];
    for (int i = p1; i < ra->k; i++) cb[kb++] = ra->c[i];
    out[0] = (plan_t){(int)mv->r1, ra->dep, rb->arr, ka, ca};
    out[1] = (plan_t){(int)mv->r2, rb->dep, ra->arr, kb, cb};
    return 2;
  }
  case DEPOT_INSERT: {
    int *ca = (int *)malloc(sizeof(int) * (size_t)(ra->k + 1)), ka = 0;
    int *cb = (int *)malloc(sizeof(int) * (size_t)(ra->k + 1)), kb = 0;
    for (int i = 0; i < p1; i++) ca[ka++] = ra->c[i];
    for (int i = p1; i < ra->k; i++) cb[kb++] = ra->c[i];
    out[0] = (plan_t){(int)mv->r1, ra->dep, ra->arr, ka, ca};
    out[1] = (plan_t){-1, (int)mv->depot, (int)mv->depot, kb, cb};
    return 2;
  }
  case DEPOT_REPLACE: {
    int dep = (mv->mode == MODE_DEPART || mv->mode == MODE_BOTH) ? (int)mv->depot : ra->dep;
    int arr = (mv->mode == MODE_ARRIVE || mv->mode == MODE_BOTH) ? (int)mv->depot : ra->arr;
    int *c = (int *)malloc(sizeof(int) * (size_t)(ra->k + 1));
    for (int i = 0; i < ra->k; i++) c[i] = ra->c[i];
    out[0] = (plan_t){(int)mv->r1, dep, arr, ra->k, c};
    return 1;
  }
  }
  return -1;
}

/* returns 0, or 2 when the move set conflicts (ValueError in the reference) */
static int apply_moves(sol_t *s, int op, const cand_t *mv, int nm) {
  /* conflict check (localsearch.py:60-65) */
  char *used = (char *)calloc((size_t)s->m + 1, 1);
  for (int i = 0; i < nm; i++) {
    int r1 = (int)mv[i].r1, r2 = (int)mv[i].r2;
    if (used[r1] || (r2 >= 0 && used[r2])) { free(used); return 2; }
    used[r1] = 1;
    if (r2 >= 0) used[r2] = 1;
  }
  free(used);
  plan_t *plans = (plan_t *)malloc(sizeof(plan_t) * (size_t)(2 * nm + 1));
  int np_ = 0;
  for (int i = 0; i < nm; i++) np_ += plan_move(s, op, &mv[i], plans + np_);
  int n_new = 0;
  for (int i = 0; i < np_; i++)
    if (plans[i].idx < 0 && plans[i].k > 0) n_new++;
  int m0 = s->m;
  sol_reserve(s, m0 + n_new);
  int at = m0;
  for (int i = 0; i < np_; i++) {
    plan_t *p = &plans[i];
    if (p->idx >= 0) route_set(&s->r[p->idx], p->dep, p->arr, p->c, p->k);
    else if (p->k > 0) route_set(&s->r[at++], p->dep, p->arr, p->c, p->k);
    free(p->c);
  }
  s->m = at;
  free(plans);
  /* drop_empty_routes (model.py:198-199), stable */
  int w = 0;
  for (int r = 0; r < s->m; r++) {
    if (s->r[r].k > 0) {
      if (w != r) { route_t t = s->r[w]; s->r[w] = s->r[r]; s->r[r] = t; }
      w++;
    }
  }
  s->m = w;
  return 0;
}

/* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src) */
static double pairwise_sum(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
  }
}

static void cache_totals(const cache_t *C, double out[5]) {
  out[0] = pairwise_sum(C->rD, C->m);
  out[1] = pairwise_sum(C->rV1, C->m);
  out[2] = pairwise_sum(C->rV2, C->m);
  out[3] = pairwise_sum(C->rV3, C->m);
  out[4] = C->I->theta * (pairwise_sum(C->rclo, C->m) + C->fexcess);
}

/* ------------------------------------------------------------------------- */
/* public API                                                                */
/* ------------------------------------------------------------------------- */
int64_t orc_count(const orc_instance_desc *inst, const orc_flat_sol *fs, int32_t op) {
  sol_t s;
  sol_from_flat(&s, fs);
  cache_t C;
  cache_build(&C, inst, &s);
  emit_t E = {NULL, 0, 0, 0};
  enum_op(&C, op, &E);
  cache_free(&C);
  sol_free(&s);
  return E.n;
}

int64_t orc_enumerate(const orc_instance_desc *inst, const orc_flat_sol *fs, int32_t op, orc_cands *cs,
                      int64_t cap) {
  sol_t s;
  sol_from_flat(&s, fs);
  cache_t C;
  cache_build(&C, inst, &s);
  emit_t E = {cs, cap, 0, 0};
  enum_op(&C, op, &E);
  cache_free(&C);
  sol_free(&s);
  if (E.overflow) return -1;
  cs->n = E.n;
  return E.n;
}

static inline cand_t cand_at(const orc_cands *cs, int64_t i) {
  cand_t c = {cs->r1[i], cs->p1[i], cs->r2[i], cs->p2[i], cs->len1[i], cs->len2[i],
              cs->depot[i], cs->mode[i], cs->rev1[i], cs->rev2[i]};
  return c;
}

int orc_evaluate(const orc_instance_desc *inst, const orc_flat_sol *fs, int32_t op, const orc_cands *cs,
                 const double lam[4], orc_deltas *out) {
  if (op < 0 || op > 5) return 1;
  sol_t s;
  sol_from_flat(&s, fs);
  cache_t C;
  cache_build(&C, inst, &s);
  for (int64_t i = 0; i < cs->n; i++) {
    cand_t c = cand_at(cs, i);
    double o[6];
    eval_one(&C, op, &c, lam, o, &out->fleet_neutral[i]);
    out->dD[i] = o[0]; out->dV1[i] = o[1]; out->dV2[i] = o[2]; out->dV3[i] = o[3];
    out->dV4[i] = o[4]; out->dF[i] = o[5];
  }
  cache_free(&C);
  sol_free(&s);
  return 0;
}

void orc_totals(const orc_instance_desc *inst, const orc_flat_sol *fs, double out[5]) {
  sol_t s;
  sol_from_flat(&s, fs);
  cache_t C;
  cache_build(&C, inst, &s);
  cache_totals(&C, out);
  cache_free(&C);
  sol_free(&s);
}

typedef struct {
  orc_cands cs;
  orc_deltas d;
  int64_t cap;
  int64_t *fol;
} work_t;

static void work_reserve(work_t *W, int64_t n) {
  if (W->cap >= n) return;
  int64_t c = n + n / 2 + 1024;
#define RA(P, T) P = (T *)realloc(P, sizeof(T) * (size_t)c)
  RA(W->cs.r1, int64_t); RA(W->cs.p1, int64_t); RA(W->cs.r2, int64_t); RA(W->cs.p2, int64_t);
  RA(W->cs.len1, int64_t); RA(W->cs.len2, int64_t); RA(W->cs.depot, int64_t); RA(W->cs.mode, int64_t);
  RA(W->cs.rev1, uint8_t); RA(W->cs.rev2, uint8_t);
  RA(W->d.dD, double); RA(W->d.dV1, double); RA(W->d.dV2, double); RA(W->d.dV3, double);
  RA(W->d.dV4, double); RA(W->d.dF, double); RA(W->d.fleet_neutral, uint8_t); RA(W->fol, int64_t);
#undef RA
  W->cap = c;
}

static void work_free(work_t *W) {
  free(W->cs.r1); free(W->cs.p1); free(W->cs.r2); free(W->cs.p2); free(W->cs.len1); free(W->cs.len2);
  free(W->cs.depot); free(W->cs.mode); free(W->cs.rev1); free(W->cs.rev2);
  free(W->d.dD); free(W->d.dV1); free(W->d.dV2); free(W->d.dV3); free(W->d.dV4); free(W->d.dF);
  free(W->d.fleet_neutral); free(W->fol);
  memset(W, 0, sizeof(*W));
}

/* enumerate + evaluate one op on a built cache into W; returns count */
static int64_t eval_op_cache(const cache_t *C, int op, const double lam[4], work_t *W) {
  emit_t E0 = {NULL, 0, 0, 0};
  enum_op(C, op, &E0);
  work_reserve(W, E0.n);
  emit_t E = {&W->cs, W->cap, 0, 0};
  enum_op(C, op, &E);
  W->cs.n = E.n;
  for (int64_t i = 0; i < E.n; i++) {
    cand_t c = cand_at(&W->cs, i);
    double o[6];
    eval_one(C, op, &c, lam, o, &W->d.fleet_neutral[i]);
    W->d.dD[i] = o[0]; W->d.dV1[i] = o[1]; W->d.dV2[i] = o[2]; W->d.dV3[i] = o[3];
    W->d.dV4[i] = o[4]; W->d.dF[i] = o[5];
  }
  return E.n;
}

static int ls_core(const orc_instance_desc *I, sol_t *s, double lam[4], const orc_ls_cfg *cfg,
                   orc_ls_stats *st, orc_ls_trace *tr) {
  memset(st, 0, sizeof(*st));
  st->best_feasible_D = INFINITY;
  if (tr && tr->snap_m) *tr->snap_m = -1;
  work_t W;
  memset(&W, 0, sizeof(W));
  cache_t C;
  cache_build(&C, I, s);
  int accepted = 0, pass = 0, rc = 0;
  for (;;) {
    if (pass >= cfg->max_passes) { rc = 5; break; } /* permutation stream exhausted */
    const int32_t *order = cfg->perms + (size_t)pass * cfg->n_ops;
    pass++;
    st->passes = pass;
    int any = 0, stop = 0;
    for (int oi = 0; oi < cfg->n_ops; oi++) {
      int op = order[oi];
      int64_t n = eval_op_cache(&C, op, lam, &W);
      st->op_evals++;
      st->cands[op] += n;
      int64_t nf = 0;
      int64_t best = orc_leader_followers(&W.cs, &W.d, cfg->multi_move, W.fol, &nf);
      if (best < 0) continue;
      /* select_moves (localsearch.py:45-55) */
      cand_t *chosen = (cand_t *)malloc(sizeof(cand_t) * (size_t)(C.m + 2));
      char *usedr = (char *)calloc((size_t)C.m + 1, 1);
      int nch = 0;
      chosen[nch++] = cand_at(&W.cs, best);
      usedr[chosen[0].r1] = 1;
      if (chosen[0].r2 >= 0) usedr[chosen[0].r2] = 1;
      if (cfg->multi_move) {
        for (int64_t f = 0; f < nf; f++) {
          cand_t c = cand_at(&W.cs, W.fol[f]);
          if (usedr[c.r1] || (c.r2 >= 0 && usedr[c.r2])) continue;
          chosen[nch++] = c;
          usedr[c.r1] = 1;
          if (c.r2 >= 0) usedr[c.r2] = 1;
        }
      }
      free(usedr);
      int arc = apply_moves(s, op, chosen, nch);
      free(chosen);
      if (arc) { rc = arc; stop = 1; break; }
      st->moves_applied += nch;
      cache_free(&C);
      cache_build(&C, I, s);
      double tot[5];
      cache_totals(&C, tot);
      int feas = 1;
      for (int i = 0; i < 4; i++) {
        /* adapt_penalties (evaluation.py:153-161) */
        int viol = tot[i + 1] > VIOLATION_TOL;
        if (viol) { lam[i] = lam[i] / cfg->kappa; feas = 0; }
        else lam[i] = lam[i] * cfg->kappa;
        double lo = cfg->lam_min, hi = cfg->lam_max;
        double x = lo > lam[i] ? lo : lam[i]; /* Python max(lam, lo) */
        lam[i] = hi < x ? hi : x;             /* Python min(x, hi) */
      }
      if (tr && accepted < tr->cap) {
        tr->op[accepted] = op;
        tr->n_moves[accepted] = nch;
        for (int i = 0; i < 4; i++) tr->lam[accepted * 4 + i] = lam[i];
        tr->D[accepted] = tot[0];
        tr->feasible[accepted] = (uint8_t)feas;
      }
      if (feas) {
        st->n_feasible++;
        if (tot[0] < st->best_feasible_D) {
          st->best_feasible_D = tot[0];
          if (tr && tr->snap_m) { /* snapshot of the new best feasible state */
            int64_t nc = 0;
            for (int r = 0; r < s->m; r++) nc += s->r[r].k;
            if (s->m <= tr->snap_cap_routes && nc <= tr->snap_cap_cust) {
              *tr->snap_m = s->m;
              tr->snap_off[0] = 0;
              for (int r = 0; r < s->m; r++) {
                tr->snap_dep[r] = s->r[r].dep;
                tr->snap_arr[r] = s->r[r].arr;
                memcpy(tr->snap_cust + tr->snap_off[r], s->r[r].c, sizeof(int32_t) * (size_t)s->r[r].k);
                tr->snap_off[r + 1] = tr->snap_off[r] + s->r[r].k;
              }
            }
          }
        }
      }
      accepted++;
      any = 1;
      st->accepted = accepted;
      if (accepted >= cfg->depth) { stop = 1; break; }
    }
    if (stop || !any) break;
  }
  st->status = rc;
  cache_free(&C);
  work_free(&W);
  return rc;
}

int orc_local_search(const orc_instance_desc *inst, const orc_flat_sol *fs, double lam[4],
                     const orc_ls_cfg *cfg, int32_t cap_routes, int32_t cap_cust, int32_t *out_m,
                     int32_t *out_off, int32_t *out_cust, int32_t *out_depart, int32_t *out_arrive,
                     orc_ls_stats *stats, orc_ls_trace *trace) {
  sol_t s;
  sol_from_flat(&s, fs);
  int rc = ls_core(inst, &s, lam, cfg, stats, trace);
  if (s.m > cap_routes) { sol_free(&s); return 3; }
  int64_t tot = 0;
  for (int r = 0; r < s.m; r++) tot += s.r[r].k;
  if (tot > cap_cust) { sol_free(&s); return 3; }
  *out_m = s.m;
  out_off[0] = 0;
  for (int r = 0; r < s.m; r++) {
    out_depart[r] = s.r[r].dep;
    out_arrive[r] = s.r[r].arr;
    memcpy(out_cust + out_off[r], s.r[r].c, sizeof(int32_t) * (size_t)s.r[r].k);
    out_off[r + 1] = out_off[r] + s.r[r].k;
  }
  sol_free(&s);
  return rc;
}

/* ---- multi-threaded drivers for the CPU baseline ------------------------- */
typedef struct {
  const orc_instance_desc *I;
  int B;
  const orc_flat_sol *sols;
  double *lam;
  const orc_ls_cfg *cfgs;
  orc_ls_stats *stats;
  orc_sol_out *outs; /* optional: final routes per individual */
  int next;
  pthread_mutex_t mu;
  /* eval-only mode */
  int eval_only;
  int64_t total;
  double checksum;
} pool_t;

static void *pool_worker(void *arg) {
  pool_t *P = (pool_t *)arg;
  work_t W;
  memset(&W, 0, sizeof(W));
  for (;;) {
    pthread_mutex_lock(&P->mu);
    int b = P->next++;
    pthread_mutex_unlock(&P->mu);
    if (b >= P->B) break;
    sol_t s;
    sol_from_flat(&s, &P->sols[b]);
    if (P->eval_only) {
      cache_t C;
      cache_build(&C, P->I, &s);
      int64_t tot = 0;
      double cs = 0.0;
      for (int op = 0; op < 6; op++) {
        if (op == TWO_OPT && P->I->has_windows) continue;
        int64_t n = eval_op_cache(&C, op, P->lam + 4 * b, &W);
        tot += n;
        for (int64_t i = 0; i < n; i++) cs += W.d.dF[i] < 0 ? W.d.dF[i] : 0.0;
      }
      cache_free(&C);
      pthread_mutex_lock(&P->mu);
      P->total += tot;
      P->checksum += cs;
      pthread_mutex_unlock(&P->mu);
    } else {
      ls_core(P->I, &s, P->lam + 4 * b, &P->cfgs[b], &P->stats[b], NULL);
      if (P->outs) {
        orc_sol_out *o = &P->outs[b];
        int64_t tot = 0;
        for (int r = 0; r < s.m; r++) tot += s.r[r].k;
        o->m = s.m;
        if (s.m > o->cap_routes || tot > o->cap_cust) {
          o->status = 3;
        } else {
          o->status = 0;
          o->off[0] = 0;
          for (int r = 0; r < s.m; r++) {
            o->depart[r] = s.r[r].dep;
            o->arrive[r] = s.r[r].arr;
            memcpy(o->cust + o->off[r], s.r[r].c, sizeof(int32_t) * (size_t)s.r[r].k);
            o->off[r + 1] = o->off[r] + s.r[r].k;
          }
        }
      }
    }
    sol_free(&s);
  }
  work_free(&W);
  return NULL;
}

static void pool_run(pool_t *P, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  pthread_mutex_init(&P->mu, NULL);
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, pool_worker, P);
  for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&P->mu);
}

int orc_local_search_many(const orc_instance_desc *inst, int32_t B, const orc_flat_sol *sols, double *lam,
                          const orc_ls_cfg *cfgs, int32_t nthreads, orc_ls_stats *stats) {
  pool_t P;
  memset(&P, 0, sizeof(P));
  P.I = inst; P.B = B; P.sols = sols; P.lam = lam; P.cfgs = cfgs; P.stats = stats;
  pool_run(&P, nthreads);
  return 0;
}

int orc_local_search_many_out(const orc_instance_desc *inst, int32_t B, const orc_flat_sol *sols, double *lam,
                              const orc_ls_cfg *cfgs, int32_t nthreads, orc_ls_stats *stats, orc_sol_out *outs) {
  pool_t P;
  memset(&P, 0, sizeof(P));
  P.I = inst; P.B = B; P.sols = sols; P.lam = lam; P.cfgs = cfgs; P.stats = stats; P.outs = outs;
  pool_run(&P, nthreads);
  for (int b = 0; b < B; b++)
    if (outs[b].status) return 3;
  return 0;
}

int64_t orc_eval_all_many(const orc_instance_desc *inst, int32_t B, const orc_flat_sol *sols,
                          const double *lam, int32_t nthreads, double *checksum) {
  pool_t P;
  memset(&P, 0, sizeof(P));
  P.I = inst; P.B = B; P.sols = sols; P.lam = (double *)lam; P.eval_only = 1;
  pool_run(&P, nthreads);
  if (checksum) *checksum = P.checksum;
  return P.total;
}
