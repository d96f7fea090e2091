/*
 * mdr_sm100.h -- C-ABI of libmdr_sm100.so, the B200 (sm_100a) implementation
 * of the reference's batched local search (mdroute, arxiv 2605.05208).
 *
 * The reference is pure Python; its "FFI" for this path is its Python API.
 * Each entry point below replaces one reference interface (file:line under
 * /root/reference/pkg/src/mdroute/); the Python package
 * paper_2605_05208_b200 binds them with ctypes and re-exposes the reference
 * signatures (INTEGRATION.md shows the binding).
 *
 *   mdr_instance_create   Instance + ScalingConstants + NeighborLists upload
 *                         (model.py:39-154, evaluation.py:109-132, neighborhood.py:45-57)
 *   mdr_pop_create/upload SolutionCache per individual (batch.py:48-158),
 *                         SolutionIndex (moves.py:151-171)
 *   mdr_count/enumerate   enumerate_candidates (moves.py:444-464)
 *   mdr_evaluate          evaluate_candidates (batch.py:365-553)
 *   mdr_leader_followers  leader_and_followers (batch.py:578-614)
 *   mdr_totals            SolutionCache.totals (batch.py:161-165)
 *   mdr_local_search      local_search (localsearch.py:97-140), population-batched:
 *                         B independent descents advance together on the device
 *   mdr_repair            repair_insert FBI/IBI/FRI/IRI (genetic.py:174-244), batched
 *   mdr_pop_breakdown     evaluate (evaluation.py:206-224) of every individual
 *   mdr_neighbor_build    neighborhood.build (neighborhood.py:60-101)
 *   mdr_shuffle_stream    the rng.shuffle calls of local_search (localsearch.py:112-113)
 *   mdr_probe_*           diagnostics: measured L2 / FP64 roofline denominators
 *
 * Conventions: plain pointers and sizes, host buffers unless stated, return
 * int status (MDR_OK ...), no C++ exceptions cross the ABI, a handle is used
 * from one host thread at a time.  `stream` is a cudaStream_t (NULL = legacy
 * default stream).  There is no CPU fallback: without a CUDA device every
 * call fails with MDR_ERR_CUDA.
 */
#ifndef MDR_SM100_H
#define MDR_SM100_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDR_OK 0
#define MDR_ERR_ARG 1      /* invalid argument (ValueError in the reference)      */
#define MDR_ERR_CONFLICT 2 /* conflicting move set (localsearch.py:63-64)         */
#define MDR_ERR_CAPACITY 3 /* route/position/follower capacity exceeded: caller
                              re-creates the population with larger caps and retries */
#define MDR_ERR_CUDA 4     /* CUDA error or no device                              */
#define MDR_ERR_PERMS 5    /* operator-permutation stream exhausted                */

/* operator codes = moves.Op (moves.py:24-30) */
#define MDR_RELOCATE 0
#define MDR_SWAP 1
#define MDR_TWO_OPT_STAR 2
#define MDR_TWO_OPT 3
#define MDR_DEPOT_INSERT 4
#define MDR_DEPOT_REPLACE 5

typedef struct mdr_instance mdr_instance;
typedef struct mdr_pop mdr_pop;

typedef struct mdr_instance_desc {
  int32_t n_nodes, n_depots;
  const double *dist, *time; /* [n*n] row-major; time == dist means "time is dist" */
  const double *demand, *service, *tw_early, *tw_late; /* [n] */
  double capacity, max_duration, fleet_per_depot;     /* +inf allowed */
  int32_t open_routes, has_windows;
  double gamma, theta;   /* ScalingConstants */
  const int32_t *lists;  /* [n * width] NeighborLists.lists, -1 padded */
  int32_t width;
} mdr_instance_desc;

/* candidate SoA in moves._FIELDS order (moves.py:174-176) */
typedef struct mdr_cands {
  int64_t n;
  int64_t *r1, *p1, *r2, *p2, *len1, *len2, *depot, *mode;
  uint8_t *rev1, *rev2;
} mdr_cands;

typedef struct mdr_deltas {
  double *dD, *dV1, *dV2, *dV3, *dV4, *dF;
  uint8_t *fleet_neutral;
} mdr_deltas;

typedef struct mdr_ls_cfg {
  int32_t depth, multi_move;       /* SearchConfig (localsearch.py:24-31) */
  double kappa, lam_min, lam_max;  /* PenaltyState (evaluation.py:135-150) */
  int32_t max_passes, n_ops;
  const uint8_t *perms;            /* [B][max_passes][n_ops]: rng.shuffle results, host */
  double deadline_s;               /* <0: none; else seconds from the call (checked between rounds) */
  int32_t rounds_per_sync;         /* device rounds per host poll (0 = default, 16) */
  int32_t use_graph;               /* reserved (graphs are used unless MDR_NO_GRAPH is set) */
  int32_t snapshot_best;           /* keep the best feasible state for mdr_pop_download_best */
  int32_t trace;                   /* record every accepted step (mdr_pop_trace) */
} mdr_ls_cfg;

typedef struct mdr_ls_stats {
  int32_t passes, accepted, op_evals, status;
  int64_t cands[6];       /* candidates scored per operator (duplicates included) */
  int64_t moves_applied;
  int32_t n_feasible;     /* feasible post-step states */
  int32_t n_improving;    /* feasible states that lowered the running minimum D */
  double best_feasible_D; /* +inf if none */
  /* on MDR_ERR_CAPACITY: the capacities a retry needs (0 = not the cause) */
  int32_t need_followers, need_queue, need_routes, need_positions;
} mdr_ls_stats;

typedef struct mdr_timing {
  double eval_ms, select_ms, plan_ms, total_ms; /* summed CUDA-event times */
  int64_t eval_launches, rounds;
  int64_t cands_total;
  double geval_ms; /* generic-path evaluator after the evaluators (intra-route, 2-opt, depot
                      operators; 0 when the population is small enough that these are
                      drained on the evaluators' graph branches, inside eval_ms) */
  /* profiling pass only: the evaluation phase serialised on one stream, per part:
   * [0] relocate staged evaluator, [1] its intra-route drain (k_eval_g region 1),
   * [2] swap, [3] its drain, [4] 2-opt*, [5] depot (+2-opt) enumerators and region-0 drain */
  double kern_ms[6];
  int64_t kern_rounds;
} mdr_timing;

const char *mdr_last_error(void);
int mdr_device_count(void);
const char *mdr_build_info(void);

int mdr_instance_create(const mdr_instance_desc *desc, int32_t device, mdr_instance **out);
void mdr_instance_destroy(mdr_instance *inst);

/* B_cap individuals, at most J_cap routes and K_cap customers per route,
 * F_cap follower entries per individual per operator evaluation. */
int mdr_pop_create(mdr_instance *inst, int32_t B_cap, int32_t J_cap, int32_t K_cap, int32_t F_cap,
                   mdr_pop **out);
void mdr_pop_destroy(mdr_pop *pop);

/* Solutions of B individuals: individual b owns routes rbase[b]..rbase[b+1]-1;
 * route r has customers cust[coff[r]..coff[r+1]), endpoints dep[r], arr[r].
 * lam: [B*4]. Builds all tables on the device. */
int mdr_pop_upload(mdr_pop *pop, int32_t B, const int32_t *rbase, const int32_t *coff,
                   const int32_t *cust, const int32_t *dep, const int32_t *arr, const double *lam,
                   void *stream);
/* inverse of upload; capacities in *n_routes / *n_cust on input, sizes on output */
int mdr_pop_download(mdr_pop *pop, int32_t *rbase, int32_t *coff, int32_t *cust, int32_t *dep,
                     int32_t *arr, double *lam, int32_t *n_routes, int32_t *n_cust, void *stream);
/* best feasible snapshot per individual (routes when D improved); same layout */
/* individuals b0 .. b0+nb-1 only (e.g. one elite for the exchange), same layout
 * as mdr_pop_download with rbase [nb+1] */
int mdr_pop_download_range(mdr_pop *pop, int32_t b0, int32_t nb, int32_t *rbase, int32_t *coff, int32_t *cust,
                           int32_t *dep, int32_t *arr, int32_t *n_routes, int32_t *n_cust, void *stream);
int mdr_pop_download_best(mdr_pop *pop, int32_t *rbase, int32_t *coff, int32_t *cust, int32_t *dep,
                          int32_t *arr, double *bestD, int32_t *n_routes, int32_t *n_cust,
                          void *stream);

int64_t mdr_count(mdr_pop *pop, int32_t b, int32_t op);
/* out->n holds the capacity on input and the count on output */
int mdr_enumerate(mdr_pop *pop, int32_t b, int32_t op, mdr_cands *out);
int mdr_evaluate(mdr_pop *pop, int32_t b, int32_t op, const mdr_cands *cs, const double lam[4],
                 mdr_deltas *out);
/* leader index (-1 if none); followers sorted by (dF, key, index) */
int mdr_leader_followers(mdr_pop *pop, const mdr_cands *cs, const mdr_deltas *d, int32_t multi_move,
                         int64_t *leader, int64_t *followers, int64_t *n_followers);
int mdr_totals(mdr_pop *pop, int32_t b, double out[5]);

/* B_active = individuals 0..B-1 of the last upload. stats: [B] */
int mdr_local_search(mdr_pop *pop, const mdr_ls_cfg *cfg, mdr_ls_stats *stats, void *stream);
int mdr_get_timing(mdr_pop *pop, mdr_timing *out);
/* The accepted steps of individual b's last traced descent (cfg.trace): per step
 * {op << 56 | feasible << 55 | n_moves, bits of the post-step distance D, n_moves packed move
 * keys (Move.key order) in selection order}.  *n = words recorded; MDR_ERR_CAPACITY if the
 * trace overflowed or out is shorter than *n.  Lets the host replay every post-step state
 * for on_feasible (localsearch.py:133-134). */
int mdr_pop_trace(mdr_pop *pop, int32_t b, uint64_t *out, int64_t cap, int64_t *n);
/* route_attr (evaluation.py:97-106) of every route of individuals b0 .. b0+nb-1 (the Route.attr
 * caches apply_moves refreshes, localsearch.py:73-80): out[((b-b0)*J_cap + r)*6 ..] =
 * {dist, load, T, E, L, TW} of the left fold with Python max/min semantics. */
int mdr_pop_route_attrs(mdr_pop *pop, int32_t b0, int32_t nb, double *out, void *stream);

/* n_passes results of CPython random.Random.shuffle(list(items)) continuing the
 * MT19937 state of rng.getstate()[1] (624 words + index, advanced in place);
 * out: [n_passes * n_items] or NULL (only advance).  Host-only; no GPU needed.
 * Replaces the rng.shuffle calls of localsearch.py:112-113. */
int mdr_shuffle_stream(uint32_t *state, int32_t n_items, const uint8_t *items, int32_t n_passes, uint8_t *out);
int mdr_set_profiling(mdr_pop *pop, int32_t on);
/* Population management of the generation loop.
 * n members; member i's edge set = edge_keys[edge_off[i] .. edge_off[i+1]), sorted unique
 * int64 keys a*N+b with a <= b (model.py:217-228).  dist: [n*n] row-major, in/out: rows and
 * columns >= row0 are (re)computed as solution_distance (population.py:19-24), the rest is
 * kept (distances do not change while both members live).  If n > mu, survivor_selection
 * (population.py:103-116) runs on cost[i] (penalised cost) and birth[i] (unique) and writes
 * the removed indices, in removal order, to removed[0 .. n-mu).
 * Replaces Population.distance_matrix / survivor_selection (population.py:94-116). */
/* Initial solutions of B individuals (genetic.initial_solution, genetic.py:251-294):
 * order[ooff[b*ND+d] .. ooff[b*ND+d+1]) = depot d's nearest-depot members of individual b after
 * the caller's rng.shuffle; each is inserted at its feasible slot of least distance increase, else
 * in a new route (d, d) while the fleet allows, else left over: n_left[b] customers in
 * left[b*N_C ..] (insertion order).  The routes replace the population's individuals 0..B-1
 * (depot-major order); the caller repairs the leftovers (mdr_repair, IBI). */
int mdr_construct(mdr_pop *pop, int32_t B, const int32_t *ooff, const int32_t *order, int32_t *n_left, int32_t *left,
                  void *stream);

/* The route exchange of DCREX (genetic.py:343-446) for B offspring of one generation.
 * Population: M members, member m owns routes mroute[m] .. mroute[m+1]-1, route r has customers
 * cust[coff[r] .. coff[r+1]) and endpoints dep[r], arr[r].  Offspring b: main parent main_idx[b],
 * donors[b*(M-1) ..] in the order rng.shuffle left them, mt[b*625 ..] = rng.getstate()[1] after
 * those draws (the stream rng.choice continues), sigma_bounds[2b..] = diversity_bounds.  Out:
 * offspring b = member routes refs[b*J_cap .. +n_refs[b]) (in order); keep[b*C_cap + i] = 1 if the
 * i-th customer slot (route order, then position) survives _remove_redundant; its unrouted
 * customers (ascending) and sigma; mt is updated to each stream after its choice draws.
 * Replaces the exchange half of genetic.dcrex. */
int mdr_route_exchange(mdr_instance *inst, int32_t M, const int32_t *mroute, const int32_t *coff, const int32_t *cust,
                       const int32_t *dep, const int32_t *arr, int32_t B, const int32_t *main_idx,
                       const int32_t *donors, uint32_t *mt, const double *sigma_bounds, int32_t J_cap,
                       int32_t C_cap, int32_t *refs, int32_t *n_refs, int32_t *keep, int32_t *unrouted,
                       int32_t *n_unrouted, double *sigma);

/* Forward simulation of n_routes node sequences (route r = seq[off[r] .. off[r+1]), depots
 * included as Route.sequence gives them): out[r*6 ..] = {distance, load, duration, time_warp,
 * late_count, minimal duration (want_min; else = duration)}.  Replaces simulate_route /
 * minimal_duration (model.py:242-314), the per-route part of check_feasible (model.py:349-392). */
int mdr_route_sim(mdr_instance *inst, int32_t n_routes, const int32_t *off, const int32_t *seq, int32_t want_min,
                  double *out);

int mdr_population_select(int32_t device, int32_t n, int32_t row0, const int64_t *edge_off, const int64_t *edge_keys,
                          double *dist, int32_t mu, double xi, const double *cost, const int64_t *birth,
                          int32_t *removed);

/* evaluator shape the population's local search launches (diagnostic, lets the
 * parity tests assert they ran the kernels the benchmark times):
 * out = {staged evaluators on, items per CTA task, warps per CTA, B_cap} */
int mdr_pop_info(mdr_pop *pop, int32_t out[4]);

/* Repair insertion (genetic.repair_insert, genetic.py:174-244) on the device
 * for individuals 0..B-1 of the last upload: op FBI=0, IBI=1, FRI=2, IRI=3 (RI
 * only draws from the rng; it stays with the caller).  pend_off [B+1], pend:
 * the unrouted customers of each individual (any order; sorted as the
 * reference does).  lam = the uploaded penalty weights.  On MDR_OK the
 * population holds the repaired solutions, rebuilt and ready for
 * mdr_local_search / mdr_pop_download.  MDR_ERR_CAPACITY: grow J_cap / K_cap
 * to stats[b].need_j / need_k, re-upload and retry. */
typedef struct mdr_repair_stats {
  int32_t status, inserted, need_j, need_k;
  int64_t slot_evals;     /* slot evaluations performed on the device */
  int64_t ref_slot_evals; /* slot evaluations the reference's full re-scan performs */
} mdr_repair_stats;
int mdr_repair(mdr_pop *pop, int32_t op, const int32_t *pend_off, const int32_t *pend, mdr_repair_stats *stats,
               void *stream);

/* evaluation.evaluate (evaluation.py:206-224) of individuals 0..B-1 with the
 * reference's scalar semantics: out[b*6 .. +6] = {D, V1, V2, V3, V4, F}, F under
 * lam[b*4 .. +4] (NULL: the population's own lambda). */
int mdr_pop_breakdown(mdr_pop *pop, const double *lam, double *out, void *stream);

/* Granular neighbour lists on the device; replaces neighborhood.build
 * (neighborhood.py:60-101).  Host buffers: dist/time [n*n] (time NULL or ==
 * dist: alias), tw_early/tw_late/service [n]; out lists [n*theta] (-1 padded,
 * rows ascending by (eta, id)), mask [n*n] (0/1) or NULL.  kernel_ms (optional)
 * receives the build kernel's device time.  theta <= 2048. */
int mdr_neighbor_build(int32_t device, int32_t n, int32_t n_depots, const double *dist, const double *time,
                       const double *tw_early, const double *tw_late, const double *service, double gamma,
                       double alpha, double beta, int32_t theta, int32_t *lists, uint8_t *mask, float *kernel_ms);

/* Diagnostic (no reference counterpart): L2 read bandwidth in GB/s, measured
 * with L1-bypassing 16-byte loads over a `bytes` buffer read `iters` times --
 * the on-chip roofline denominator bench.py reports beside the HBM peak. */
int mdr_probe_l2_gbs(int32_t device, int64_t bytes, int32_t iters, double *gbs);
/* Diagnostic: fp64 dadd/dmul throughput in G ops/s (FMA contraction off, as in
 * the evaluators) -- the FP64-pipe roofline denominator of SURVEY.md 8(d). */
int mdr_probe_fp64_gops(int32_t device, int32_t iters, double *gops);

#ifdef __cplusplus
}
#endif
#endif
