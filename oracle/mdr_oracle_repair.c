/*
 * mdr_oracle_repair.c -- CPU restatement of the reference's repair insertion.
 *
 * TEST INFRASTRUCTURE ONLY (see mdr_oracle.h): the parity checker and CPU
 * baseline for the device repair (paper_2605_05208_b200/csrc/mdr_repair.cu).
 *
 * Restates /root/reference/pkg/src/mdroute/genetic.py literally, with the
 * reference's full re-scan of every (pending customer x slot) per insertion:
 *   evaluation.concat          evaluation.py:74-94   (Python max/min: first wins)
 *   _RouteEval                 genetic.py:71-97      pref = left fold, suf = RIGHT fold
 *   _route_cost_terms          genetic.py:100-106
 *   _attr_feasible             genetic.py:109-116
 *   InsertState.slot_delta     genetic.py:130-140
 *   InsertState.open_route     genetic.py:148-166
 *   _best_slot                 genetic.py:174-190
 *   repair_insert (FBI/IBI/FRI/IRI) genetic.py:193-244
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "mdr_oracle.h"

typedef struct {
  double dist, load, T, E, L, TW;
  int first, last;
} rattr;

/* Python's built-in max(a, b) / min(a, b): the first argument unless the second
 * compares strictly greater / smaller */
static inline double py_max(double a, double b) { return b > a ? b : a; }
static inline double py_min(double a, double b) { return b < a ? b : a; }

static rattr r_single(const orc_instance_desc *I, int v) {
  rattr a = {0.0, I->demand[v], I->service[v], I->tw_early[v], I->tw_late[v], 0.0, v, v};
  return a;
}


static rattr r_concat(const orc_instance_desc *I, rattr a, rattr b) {
  if (b.first < 0) return a;
  if (a.first < 0) return b;
  const size_t lk = (size_t)a.last * I->n_nodes + b.first;
  const double t = I->time[lk], c = I->dist[lk];
  const double delta = (a.T - a.TW) + t;
  const double wait = py_max((b.E - delta) - a.L, 0.0);
  const double warp = py_max((a.E + delta) - b.L, 0.0);
  rattr o;
  o.dist = (a.dist + c) + b.dist;
  o.load = a.load + b.load;
  o.T = ((a.T + b.T) + t) + wait;
  o.E = py_max(b.E - delta, a.E) - wait;
  o.L = py_min(b.L - delta, a.L) + warp;
  o.TW = (a.TW + b.TW) + warp;
  o.first = a.first;
  o.last = b.last;
  return o;
}

static void r_terms(const orc_instance_desc *I, rattr a, double o[4]) {
  o[0] = a.dist;
  o[1] = I->has_windows ? I->gamma * a.TW : 0.0;
  o[2] = (I->theta * py_max(a.load - I->capacity, 0.0)) / I->capacity;
  o[3] = isinf(I->max_duration) ? 0.0 : (I->theta * py_max(a.T - I->max_duration, 0.0)) / I->max_duration;
}

static int r_feasible(const orc_instance_desc *I, rattr a) {
  if (a.load > I->capacity + 1e-9) return 0;
  if (!isinf(I->max_duration) && a.T > I->max_duration + 1e-9) return 0;
  if (I->has_windows && a.TW > 1e-9) return 0;
  return 1;
}

/* working solution: route r = depart, customers, arrive; pref/suf per route */
typedef struct {
  int m, cap_r, cap_k;
  int *k, *dep, *arr, *cust; /* cust[r * cap_k + i] */
  rattr *pref, *suf;         /* [r * (cap_k + 2) + i] */
} rsol;

static int r_seq(const orc_instance_desc *I, const rsol *S, int r, int i) {
  if (i == 0) return S->dep[r];
  if (i <= S->k[r]) return S->cust[(size_t)r * S->cap_k + i - 1];
  return S->arr[r];
}

static void r_rebuild(const orc_instance_desc *I, rsol *S, int r) {
  const int n = S->k[r] + (I->open_routes ? 1 : 2), w = S->cap_k + 2;
  rattr *P = S->pref + (size_t)r * w, *Q = S->suf + (size_t)r * w;
  P[0] = r_single(I, r_seq(I, S, r, 0));
  for (int i = 1; i < n; i++) P[i] = r_concat(I, P[i - 1], r_single(I, r_seq(I, S, r, i)));
  Q[n - 1] = r_single(I, r_seq(I, S, r, n - 1));
  for (int i = n - 2; i >= 0; i--) Q[i] = r_concat(I, r_single(I, r_seq(I, S, r, i)), Q[i + 1]);
}

/* (dD, dF, feasible) of inserting node before customer index pos of route r */
static void r_slot(const orc_instance_desc *I, const rsol *S, int r, int pos, int node, const double lam[4],
                   double *dd, double *df, int *feas) {
  const int n = S->k[r] + (I->open_routes ? 1 : 2), w = S->cap_k + 2;
  const rattr *P = S->pref + (size_t)r * w, *Q = S->suf + (size_t)r * w;
  rattr a = r_concat(I, P[pos], r_single(I, node));
  if (pos + 1 < n) a = r_concat(I, a, Q[pos + 1]);
  double o[4], x[4];
  r_terms(I, P[n - 1], o);
  r_terms(I, a, x);
  *dd = x[0] - o[0];
  *df = ((*dd + lam[0] * (x[1] - o[1])) + lam[1] * (x[2] - o[2])) + lam[2] * (x[3] - o[3]);
  *feas = r_feasible(I, a);
}

/* _best_slot: first slot of minimal cost, second-smallest cost (multiset) */
static int r_best_slot(const orc_instance_desc *I, const rsol *S, int node, int feasible_only, const double lam[4],
                       int *br, int *bp, double *c1o, double *c2o, long long *evals) {
  int found = 0;
  double c1 = INFINITY, c2 = INFINITY;
  for (int r = 0; r < S->m; r++)
    for (int pos = 0; pos <= S->k[r]; pos++) {
      double dd, df;
      int feas;
      r_slot(I, S, r, pos, node, lam, &dd, &df, &feas);
      (*evals)++;
      if (feasible_only && !feas) continue;
      const double cost = feasible_only ? dd : df;
      if (cost < c1) {
        *br = r; *bp = pos; found = 1;
        c2 = c1;
        c1 = cost;
      } else if (cost < c2) {
        c2 = cost;
      }
    }
  *c1o = c1;
  *c2o = c2;
  return found;
}

static int r_open_route(const orc_instance_desc *I, rsol *S, int node) {
  if (S->m >= S->cap_r) return -1;
  int counts[4096];
  const int nd = I->n_depots;
  for (int d = 0; d < nd; d++) counts[d] = 0;
  for (int r = 0; r < S->m; r++)
    if (S->k[r] > 0) counts[S->dep[r]]++;
  int best = -1, bnf = 0;
  double bcost = 0.0;
  for (int d = 0; d < nd; d++) {
    const double cost = I->dist[(size_t)d * I->n_nodes + node] +
                        (I->open_routes ? 0.0 : I->dist[(size_t)node * I->n_nodes + d]);
    const int free_ = isinf(I->fleet_per_depot) || (double)counts[d] < I->fleet_per_depot;
    const int nf = !free_;
    /* key (not free, cost, d): lexicographic minimum, first wins */
    if (best < 0 || nf < bnf || (nf == bnf && cost < bcost)) {
      best = d; bnf = nf; bcost = cost;
    }
  }
  const int r = S->m++;
  S->k[r] = 1;
  S->dep[r] = S->arr[r] = best;
  S->cust[(size_t)r * S->cap_k] = node;
  r_rebuild(I, S, r);
  return r;
}

static int r_insert(const orc_instance_desc *I, rsol *S, int r, int pos, int node) {
  if (S->k[r] >= S->cap_k) return -1;
  int *c = S->cust + (size_t)r * S->cap_k;
  for (int i = S->k[r]; i > pos; i--) c[i] = c[i - 1];
  c[pos] = node;
  S->k[r]++;
  r_rebuild(I, S, r);
  return 0;
}

static int cmp_i32(const void *a, const void *b) {
  const int x = *(const int *)a, y = *(const int *)b;
  return (x > y) - (x < y);
}

int orc_repair(const orc_instance_desc *I, const orc_flat_sol *sol, const int32_t *pend, int32_t n_pend, int32_t op,
               const double lam[4], int32_t out_cap_routes, int32_t out_cap_cust, int32_t *out_m, int32_t *out_off,
               int32_t *out_cust, int32_t *out_depart, int32_t *out_arrive, int64_t *slot_evals) {
  if (op < 0 || op > 3) return 1;
  const int ncust_in = sol->m ? sol->off[sol->m] : 0;
  const int total = ncust_in + n_pend;
  rsol S;
  S.m = sol->m;
  S.cap_r = sol->m + n_pend;
  S.cap_k = total > 0 ? total : 1;
  S.k = calloc((size_t)S.cap_r + 1, sizeof(int));
  S.dep = calloc((size_t)S.cap_r + 1, sizeof(int));
  S.arr = calloc((size_t)S.cap_r + 1, sizeof(int));
  S.cust = calloc(((size_t)S.cap_r + 1) * S.cap_k, sizeof(int));
  S.pref = calloc(((size_t)S.cap_r + 1) * (S.cap_k + 2), sizeof(rattr));
  S.suf = calloc(((size_t)S.cap_r + 1) * (S.cap_k + 2), sizeof(rattr));
  int *pending = malloc(sizeof(int) * (n_pend + 1));
  int rc = 0;
  long long evals = 0;
  if (!S.k || !S.dep || !S.arr || !S.cust || !S.pref || !S.suf || !pending) { rc = 4; goto done; }
  for (int r = 0; r < sol->m; r++) {
    S.k[r] = sol->off[r + 1] - sol->off[r];
    S.dep[r] = sol->depart[r];
    S.arr[r] = sol->arrive[r];
    for (int i = 0; i < S.k[r]; i++) S.cust[(size_t)r * S.cap_k + i] = sol->cust[sol->off[r] + i];
    r_rebuild(I, &S, r);
  }
  for (int q = 0; q < n_pend; q++) pending[q] = pend[q];
  qsort(pending, n_pend, sizeof(int), cmp_i32);
  int np = n_pend;
  const int feasible_only = op == 0 || op == 2, regret = op == 2 || op == 3;
  if (!feasible_only && S.m == 0 && np > 0) {
    if (r_open_route(I, &S, pending[0]) < 0) { rc = 3; goto done; }
    memmove(pending, pending + 1, sizeof(int) * (np - 1));
    np--;
  }
  while (np > 0) {
    int chosen = -1, cr = -1, cp = -1;
    if (regret) {
      int bcls = 0, bnode = 0;
      double bval = 0.0;
      for (int q = 0; q < np; q++) {
        const int node = pending[q];
        int r = -1, p = -1;
        double c1, c2;
        const int found = r_best_slot(I, &S, node, feasible_only, lam, &r, &p, &c1, &c2, &evals);
        int cls;
        double val;
        if (!found) { cls = 2; val = 0.0; }
        else if (isinf(c2) && c2 > 0) { cls = 1; val = 0.0; }
        else { cls = 0; val = c2 - c1; }
        /* key (cls, val, -node) > best_key */
        const int better = chosen < 0 || cls > bcls || (cls == bcls && (val > bval || (val == bval && -node > -bnode)));
        if (better) {
          bcls = cls; bval = val; bnode = node;
          chosen = q; cr = found ? r : -1; cp = found ? p : -1;
        }
      }
    } else {
      double best_cost = INFINITY;
      for (int q = 0; q < np; q++) {
        int r = -1, p = -1;
        double c1, c2;
        const int found = r_best_slot(I, &S, pending[q], feasible_only, lam, &r, &p, &c1, &c2, &evals);
        if (found && c1 < best_cost) { best_cost = c1; chosen = q; cr = r; cp = p; }
      }
      if (chosen < 0) { chosen = 0; cr = -1; }
    }
    const int node = pending[chosen];
    memmove(pending + chosen, pending + chosen + 1, sizeof(int) * (np - chosen - 1));
    np--;
    if (cr < 0) {
      if (r_open_route(I, &S, node) < 0) { rc = 3; goto done; }
    } else if (r_insert(I, &S, cr, cp, node) < 0) {
      rc = 3;
      goto done;
    }
  }
  if (S.m > out_cap_routes) { rc = 3; goto done; }
  {
    int c = 0;
    out_off[0] = 0;
    for (int r = 0; r < S.m; r++) {
      if (c + S.k[r] > out_cap_cust) { rc = 3; goto done; }
      for (int i = 0; i < S.k[r]; i++) out_cust[c++] = S.cust[(size_t)r * S.cap_k + i];
      out_off[r + 1] = c;
      out_depart[r] = S.dep[r];
      out_arrive[r] = S.arr[r];
    }
    *out_m = S.m;
  }
done:
  if (slot_evals) *slot_evals = evals;
  free(S.k); free(S.dep); free(S.arr); free(S.cust); free(S.pref); free(S.suf); free(pending);
  return rc;
}

/* ---- many independent repairs on host threads (bench cpu baseline) ---- */
typedef struct {
  const orc_instance_desc *I;
  int B;
  const orc_flat_sol *sols;
  const int32_t *pend_off, *pend;
  int32_t op;
  const double *lam;
  int64_t *evals;
  int32_t *status;
  int next;
  pthread_mutex_t mu;
} rpool_t;

static void *rpool_worker(void *arg) {
  rpool_t *P = arg;
  for (;;) {
    pthread_mutex_lock(&P->mu);
    const int b = P->next++;
    pthread_mutex_unlock(&P->mu);
    if (b >= P->B) break;
    const orc_flat_sol *s = &P->sols[b];
    const int np = P->pend_off[b + 1] - P->pend_off[b];
    const int nc = (s->m ? s->off[s->m] : 0) + np, cr = s->m + np;
    int32_t *buf = malloc(sizeof(int32_t) * ((size_t)nc + 4 * (size_t)cr + 8));
    int32_t m = 0;
    int64_t ev = 0;
    P->status[b] = orc_repair(P->I, s, P->pend + P->pend_off[b], np, P->op, P->lam + 4 * (size_t)b, cr, nc, &m,
                              buf, buf + cr + 1, buf + cr + 1 + nc, buf + 2 * cr + 1 + nc, &ev);
    P->evals[b] = ev;
    free(buf);
  }
  return NULL;
}

int orc_repair_many(const orc_instance_desc *I, int32_t B, const orc_flat_sol *sols, const int32_t *pend_off,
                    const int32_t *pend, int32_t op, const double *lam, int32_t nthreads, int64_t *evals,
                    int32_t *status) {
  rpool_t P;
  memset(&P, 0, sizeof(P));
  P.I = I; P.B = B; P.sols = sols; P.pend_off = pend_off; P.pend = pend; P.op = op; P.lam = lam;
  P.evals = evals; P.status = status;
  pthread_mutex_init(&P.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  pthread_t *th = malloc(sizeof(pthread_t) * nthreads);
  for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, rpool_worker, &P);
  for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&P.mu);
  return 0;
}
