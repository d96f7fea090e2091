// mdr_api.cu -- host side of libmdr_sm100.so: the C-ABI of include/mdr_sm100.h.
//
// Owns all device memory (instance, population tables, round scratch) and
// drives the population-batched local search: per device round one plan,
// one fused evaluate and one select/apply launch, polled every few rounds
// for completion and the caller's deadline (localsearch.py:116-117).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mdr_sm100.h"
#include "mdr_kernels.cuh"

using namespace mdr;

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

namespace mdr {
int mdr_fail(int code, const char *msg) { return fail(code, msg); }
}  // namespace mdr

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e__ = (call);                                                             \
    if (e__ != cudaSuccess) return fail(MDR_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e__)); \
  } while (0)

struct mdr_instance {
  int device;
  DevInst I;
  std::vector<void *> allocs;
};

struct mdr_pop {
  mdr_instance *inst;
  DevPop P;
  int B;
  int grid;
  std::vector<void *> allocs;
  size_t max_chunks;
  // perms buffer
  uint8_t *d_perms;
  size_t perms_cap;
  // transfer scratch
  int *d_xfer;
  size_t xfer_cap;
  int *d_hdr;
  int *h_hdr;  // pinned
  // timing
  int profiling;
  mdr_timing tm;
  cudaEvent_t ev[8];
  std::vector<cudaEvent_t> rev;  // per-round events when profiling (5 per round)
  std::vector<cudaEvent_t> kev;  // per-round per-evaluator events when profiling (7 per round)
  cudaStream_t ls;               // private stream of the round loop (graph capture)
  cudaEvent_t join[2];
  cudaStream_t side[4];          // fork/join branches of the per-operator evaluators ([3]: relocate boundary family)
  cudaEvent_t fev[6];
  // the round-batch graph, kept across calls while the launch parameters it
  // captured (instance, population, search parameters, rounds per batch) match
  cudaGraphExec_t gx = nullptr;
  std::vector<unsigned char> gkey;
  // repair scratch (mdr_repair), grown on demand
  char *rp_pre = nullptr, *rp_suf = nullptr;
  double *rp_c1 = nullptr, *rp_c2 = nullptr;
  int *rp_p1 = nullptr, *rp_pend = nullptr, *rp_status = nullptr;
  long long *rp_stats = nullptr;
  double *rp_fold = nullptr;
  int *rp_foldi = nullptr;
  double *bd_rt = nullptr, *bd_io = nullptr;  // mdr_pop_breakdown scratch
  double *ra_buf = nullptr;                    // mdr_pop_route_attrs output (kept: a per-call
  size_t ra_cap = 0;                           // cudaMalloc/cudaFree cost up to ~0.4 s at times)
  unsigned long long *tr_buf = nullptr;        // accepted-step trace (cfg.trace)
  long long *tr_cnt = nullptr;
  size_t tr_cap[2] = {0, 0};
  long long tr_per = 0;                        // words per individual of the last traced run
  size_t rp_cap[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
};

template <typename T>
static int dalloc(std::vector<void *> &owner, T **p, size_t n) {
  if (n == 0) n = 1;
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, n * sizeof(T));
  if (e != cudaSuccess) return fail(MDR_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  owner.push_back(q);
  *p = reinterpret_cast<T *>(q);
  return MDR_OK;
}

template <typename T>
static int regrow(T **ptr, size_t &cap, size_t need) {
  if (cap >= need && *ptr) return MDR_OK;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  cap = 0;
  CK(cudaMalloc((void **)ptr, need * sizeof(T)));
  cap = need;
  return MDR_OK;
}

#define DA(owner, ptr, n)                        \
  do {                                           \
    int rc__ = dalloc(owner, &(ptr), (size_t)(n)); \
    if (rc__) return rc__;                       \
  } while (0)

extern "C" {

const char *mdr_last_error(void) { return g_err.c_str(); }

int mdr_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

const char *mdr_build_info(void) {
  return "libmdr_sm100: sm_100a (compute_100a), fp64 with -fmad=false";
}

int mdr_instance_create(const mdr_instance_desc *d, int32_t device, mdr_instance **out) {
  if (!d || !out) return fail(MDR_ERR_ARG, "null argument");
  int N = d->n_nodes, ND = d->n_depots;
  if (ND < 1 || N - ND < 1) return fail(MDR_ERR_ARG, "instance needs at least one depot and one customer");
  if (ND > 254) return fail(MDR_ERR_ARG, "at most 254 depots supported");
  if (d->width < 1) return fail(MDR_ERR_ARG, "neighbour list width must be >= 1");
  if (!d->dist || !d->demand || !d->service || !d->tw_early || !d->tw_late || !d->lists)
    return fail(MDR_ERR_ARG, "null array in instance descriptor");
  int ndev = mdr_device_count();
  if (ndev <= 0) return fail(MDR_ERR_CUDA, "no CUDA device (the sm_100a library has no CPU path)");
  if (device < 0 || device >= ndev) return fail(MDR_ERR_ARG, "bad device index");
  CK(cudaSetDevice(device));
  mdr_instance *I = new mdr_instance();
  I->device = device;
  auto bail = [&](int code, const std::string &msg) {
    for (void *q : I->allocs) cudaFree(q);
    delete I;
    return fail(code, msg);
  };
#define CKI(call)                                                                              \
  do {                                                                                         \
    cudaError_t e__ = (call);                                                                  \
    if (e__ != cudaSuccess) return bail(MDR_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e__)); \
  } while (0)
  DevInst &D = I->I;
  D.N = N; D.ND = ND; D.NC = N - ND; D.W = d->width;
  size_t nn = (size_t)N * N;
  double *dist = nullptr, *time = nullptr;
  int rc;
  if ((rc = dalloc(I->allocs, &dist, nn))) return bail(rc, g_err);
  CKI(cudaMemcpy(dist, d->dist, nn * sizeof(double), cudaMemcpyHostToDevice));
  D.talias = (d->time == nullptr || d->time == d->dist);
  if (!D.talias) {
    if ((rc = dalloc(I->allocs, &time, nn))) return bail(rc, g_err);
    CKI(cudaMemcpy(time, d->time, nn * sizeof(double), cudaMemcpyHostToDevice));
  } else {
    time = dist;
  }
  D.dist = dist; D.time = time;
  std::vector<double4> node(N);
  for (int v = 0; v < N; v++) node[v] = make_double4(d->demand[v], d->service[v], d->tw_early[v], d->tw_late[v]);
  double4 *dnode = nullptr;
  if ((rc = dalloc(I->allocs, &dnode, N))) return bail(rc, g_err);
  CKI(cudaMemcpy(dnode, node.data(), N * sizeof(double4), cudaMemcpyHostToDevice));
  D.node = dnode;
  int *lists = nullptr;
  size_t nl = (size_t)(N - ND) * d->width;
  if ((rc = dalloc(I->allocs, &lists, nl))) return bail(rc, g_err);
  CKI(cudaMemcpy(lists, d->lists + (size_t)ND * d->width, nl * sizeof(int), cudaMemcpyHostToDevice));
  D.lists = lists;
  D.Q = d->capacity; D.Dmax = d->max_duration; D.NV = d->fleet_per_depot;
  D.d_on = !std::isinf(d->max_duration);
  D.nv_on = !std::isinf(d->fleet_per_depot);
  D.open = d->open_routes ? 1 : 0;
  D.win = d->has_windows ? 1 : 0;
  D.gamma = d->gamma; D.theta = d->theta;
  D.rQ = 1.0 / d->capacity;
  {
    // exact (bitwise) symmetry of dist and time enables row-oriented link reads
    int sym = 1;
    for (int x = 0; x < N && sym; x++)
      for (int y = x + 1; y < N; y++) {
        size_t a = (size_t)x * N + y, b = (size_t)y * N + x;
        if (memcmp(&d->dist[a], &d->dist[b], 8) || (!D.talias && memcmp(&d->time[a], &d->time[b], 8))) {
          sym = 0;
          break;
        }
      }
    D.sym = getenv("MDR_NO_SYM") ? 0 : sym;
  }
  D.rD = 1.0 / d->max_duration;
  CKI(cudaDeviceSynchronize());
#undef CKI
  *out = I;
  return MDR_OK;
}

void mdr_instance_destroy(mdr_instance *I) {
  if (!I) return;
  cudaSetDevice(I->device);
  for (void *p : I->allocs) cudaFree(p);
  delete I;
}

static int pop_build(mdr_pop *p, mdr_instance *inst, int32_t Bcap, int32_t J, int32_t K, int32_t Fcap);

int mdr_pop_create(mdr_instance *inst, int32_t Bcap, int32_t J, int32_t K, int32_t Fcap, mdr_pop **out) {
  if (!inst || !out) return fail(MDR_ERR_ARG, "null argument");
  if (Bcap < 1 || J < 1 || K < 1 || Fcap < 1) return fail(MDR_ERR_ARG, "capacities must be >= 1");
  if (J > 4094) return fail(MDR_ERR_ARG, "J_cap must be <= 4094 (12-bit route field of the packed key)");
  if (K > 500) return fail(MDR_ERR_ARG, "K_cap must be <= 500 (9-bit position field of the packed key)");
  CK(cudaSetDevice(inst->device));
  mdr_pop *p = new mdr_pop();  // value-initialised: every handle starts null
  p->inst = inst;
  const int rc = pop_build(p, inst, Bcap, J, K, Fcap);
  if (rc != MDR_OK) {
    const std::string msg = g_err;
    mdr_pop_destroy(p);  // frees whatever was allocated before the failure
    return fail(rc, msg);
  }
  *out = p;
  return MDR_OK;
}

// every failure returns straight out; mdr_pop_create then releases the partial pop
static int pop_build(mdr_pop *p, mdr_instance *inst, int32_t Bcap, int32_t J, int32_t K, int32_t Fcap) {
  memset(&p->tm, 0, sizeof(p->tm));
  p->B = 0;
  DevPop &P = p->P;
  const DevInst &I = inst->I;
  P.Bcap = Bcap; P.J = J; P.K = K; P.Kp = K + 2; P.Fcap = Fcap; P.FE = I.win ? 6 : 4;
  P.N = I.N; P.ND = I.ND;
  P.staged = (J * (I.win ? 176 : 168) <= 96 * 1024) ? 1 : 0;  // RBT staging fits shared memory
  // staged-evaluator shape: the large one once the population holds >= 100k customers, or
  // >= 24k customers of instances with >= 768 (>= 24 large tasks per individual).  Measured:
  // C4 at 64 / 32 individuals +17 % / +4 % with the large shape; C2 (64 x 288) and C3 (128 x 360)
  // -22 % / -21 % with it
  const long long tot = (long long)Bcap * I.NC;
  P.ct = (tot >= 100000 || (I.NC >= 768 && tot >= 24000)) ? MDR_LARGE_CT : MDR_SMALL_CT;
  if (getenv("MDR_CT")) P.ct = atoi(getenv("MDR_CT")) == MDR_LARGE_CT ? MDR_LARGE_CT : MDR_SMALL_CT;
  // sub-tasks per customer block (MDR_TSPLIT): measured slower at every population size
  // (C4 pop 32: 17.35 / 17.10 / 16.09 G/s for 1 / 2 / 4), so 1 by default
  P.tsplit = 1;
  if (getenv("MDR_TSPLIT")) P.tsplit = std::max(1, std::min(8, atoi(getenv("MDR_TSPLIT"))));
  if (getenv("MDR_NO_STAGED")) P.staged = 0;
  auto &A = p->allocs;
  size_t rows = (size_t)Bcap * J, slots = rows * P.Kp;
  DA(A, P.m, Bcap);
  DA(A, P.rmeta, rows);
  DA(A, P.seq, slots);
  DA(A, P.loc, (size_t)Bcap * I.N);
  DA(A, P.nxs, (size_t)Bcap * I.N);
  DA(A, P.rcon, rows);
  DA(A, P.tabP, slots * P.FE);
  DA(A, P.tabS, slots * P.FE);
  DA(A, P.tabT, slots * P.Kp * P.FE);
  DA(A, P.fleet, (size_t)Bcap * I.ND);
  DA(A, P.fexcess, Bcap);
  DA(A, P.lam, (size_t)Bcap * 4);
  DA(A, P.st, Bcap);
  DA(A, P.cands, (size_t)Bcap * 6);
  DA(A, P.op_cur, Bcap);
  DA(A, P.wsize, Bcap);
  DA(A, P.chunk_off, Bcap + 1);
  DA(A, P.total_chunks, 1);
  DA(A, P.active, 1);
  long long wmax = 0;
  for (int op = 0; op < 6; op++) {
    long long w = op_items(op, J, I.NC, I.W, I.ND, I.win, I.open, K);
    if (w > wmax) wmax = w;
  }
  if (wmax > 0x7fffffffLL) return fail(MDR_ERR_ARG, "candidate index space exceeds 2^31 per individual");
  p->max_chunks = (size_t)Bcap * (size_t)(I.NC + J);  // tasks per round
  DA(A, P.partial, p->max_chunks);
  DA(A, P.tcount, p->max_chunks);
  DA(A, P.task_next, 8);  // [6]: relocate boundary family when split
  DA(A, P.opcnt, 6);
  DA(A, P.optasks, 6);
  DA(A, P.opb, (size_t)6 * Bcap);
  DA(A, P.opoff, (size_t)6 * (Bcap + 1));
  DA(A, P.leader, Bcap);
  DA(A, P.gcount, 3);
  {
    long long g = (long long)Bcap * std::max((long long)I.NC * 64, (long long)Fcap);
    if (g > 0x7fffffffLL) g = 0x7fffffffLL;
    P.Gcap = (int)g;
  }
  DA(A, P.gq, (size_t)P.Gcap);
  // region A of the generic queue (drained concurrently with the staged
  // evaluators) only when those leave the GPU under-filled
  P.gbase[0] = 0; P.gbase[1] = 0; P.gbase[2] = P.Gcap; P.gbase[3] = P.Gcap;
  // per-producer generic-queue regions, drained on the producers' graph branches
  // (C2 +7 %, C4 +1.3 %, C5 +1 % over one queue drained after all evaluators)
  if (P.staged && !getenv("MDR_NO_OVERLAP")) {
    P.gbase[1] = P.Gcap / 3;
    P.gbase[2] = 2 * (P.Gcap / 3);
  }
  DA(A, P.fol, (size_t)Bcap * Fcap);
  DA(A, P.fcount, Bcap);
  DA(A, P.nanflag, Bcap);
  DA(A, P.scratch_seq, slots);
  DA(A, P.scratch_meta, rows);
  DA(A, P.best_m, Bcap);
  DA(A, P.best_meta, rows);
  DA(A, P.best_seq, slots);
  CK(cudaMemset(P.m, 0, sizeof(int) * Bcap));
  CK(cudaMemset(P.nxs, 0xff, sizeof(int) * (size_t)Bcap * I.N));
  CK(cudaMemset(P.best_m, 0, sizeof(int) * Bcap));
  CK(cudaMemset(P.rmeta, 0, sizeof(int4) * rows));
  CK(cudaMemset(P.st, 0, sizeof(LsState) * Bcap));
  CK(cudaMemset(P.cands, 0, sizeof(unsigned long long) * Bcap * 6));
  P.perms = nullptr; P.maxp = 0; P.nops = 0;
  p->d_perms = nullptr; p->perms_cap = 0;
  p->d_xfer = nullptr; p->xfer_cap = 0;
  DA(A, p->d_hdr, 4);
  CK(cudaMallocHost(&p->h_hdr, 4 * sizeof(int)));
  p->grid = eval_grid_size(I.win);
  p->profiling = 0;
  for (int i = 0; i < 8; i++) CK(cudaEventCreate(&p->ev[i]));
  CK(cudaStreamCreateWithFlags(&p->ls, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&p->join[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&p->join[1], cudaEventDisableTiming));
  for (int q = 0; q < 4; q++) CK(cudaStreamCreateWithFlags(&p->side[q], cudaStreamNonBlocking));
  for (int q = 0; q < 6; q++) CK(cudaEventCreateWithFlags(&p->fev[q], cudaEventDisableTiming));
  return MDR_OK;
}

void mdr_pop_destroy(mdr_pop *p) {
  if (!p) return;
  cudaSetDevice(p->inst->device);
  if (p->gx) cudaGraphExecDestroy(p->gx);
  for (void *q : p->allocs) cudaFree(q);
  if (p->d_perms) cudaFree(p->d_perms);
  if (p->d_xfer) cudaFree(p->d_xfer);
  if (p->h_hdr) cudaFreeHost(p->h_hdr);
  for (int i = 0; i < 8; i++)
    if (p->ev[i]) cudaEventDestroy(p->ev[i]);
  for (cudaEvent_t e : p->rev) cudaEventDestroy(e);
  for (cudaEvent_t e : p->kev) cudaEventDestroy(e);
  if (p->ls) cudaStreamDestroy(p->ls);
  for (int q = 0; q < 2; q++)
    if (p->join[q]) cudaEventDestroy(p->join[q]);
  for (int q = 0; q < 4; q++)
    if (p->side[q]) cudaStreamDestroy(p->side[q]);
  for (int q = 0; q < 6; q++)
    if (p->fev[q]) cudaEventDestroy(p->fev[q]);
  if (p->tr_buf) cudaFree(p->tr_buf);
  if (p->ra_buf) cudaFree(p->ra_buf);
  if (p->tr_cnt) cudaFree(p->tr_cnt);
  for (void *q : {(void *)p->rp_pre, (void *)p->rp_suf, (void *)p->rp_c1, (void *)p->rp_c2, (void *)p->rp_p1, (void *)p->rp_pend,
                  (void *)p->rp_status, (void *)p->rp_stats, (void *)p->rp_fold, (void *)p->rp_foldi,
                  (void *)p->bd_rt, (void *)p->bd_io})
    if (q) cudaFree(q);
  delete p;
}

static int ensure_xfer(mdr_pop *p, size_t n) {
  if (p->xfer_cap >= n) return MDR_OK;
  if (p->d_xfer) cudaFree(p->d_xfer);
  p->d_xfer = nullptr;
  size_t c = n + n / 2 + 1024;
  CK(cudaMalloc(&p->d_xfer, c * sizeof(int)));
  p->xfer_cap = c;
  return MDR_OK;
}

int mdr_pop_upload(mdr_pop *p, int32_t B, const int32_t *rbase, const int32_t *coff, const int32_t *cust,
                   const int32_t *dep, const int32_t *arr, const double *lam, void *stream) {
  if (!p || B < 0 || B > p->P.Bcap) return fail(MDR_ERR_ARG, "B out of range");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(p->inst->device));
  const DevInst &I = p->inst->I;
  int R = rbase[B];
  int C = coff[R];
  for (int b = 0; b < B; b++) {
    int m = rbase[b + 1] - rbase[b];
    if (m < 0) return fail(MDR_ERR_ARG, "rbase must be non-decreasing");
    if (m > p->P.J) return fail(MDR_ERR_CAPACITY, "individual has more routes than J_cap");
  }
  for (int r = 0; r < R; r++) {
    int k = coff[r + 1] - coff[r];
    if (k < 0) return fail(MDR_ERR_ARG, "coff must be non-decreasing");
    if (k > p->P.K) return fail(MDR_ERR_CAPACITY, "route longer than K_cap");
    if (dep[r] < 0 || dep[r] >= I.ND || arr[r] < 0 || arr[r] >= I.ND)
      return fail(MDR_ERR_ARG, "route endpoint is not a depot");
  }
  for (int c = 0; c < C; c++)
    if (cust[c] < I.ND || cust[c] >= I.N) return fail(MDR_ERR_ARG, "customer id out of range");
  size_t need = (size_t)(B + 1) + (R + 1) + C + 2 * (size_t)R;
  int rc = ensure_xfer(p, need);
  if (rc) return rc;
  int *d_rbase = p->d_xfer, *d_coff = d_rbase + B + 1, *d_cust = d_coff + R + 1, *d_dep = d_cust + C,
      *d_arr = d_dep + R;
  CK(cudaMemcpyAsync(d_rbase, rbase, sizeof(int) * (B + 1), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_coff, coff, sizeof(int) * (R + 1), cudaMemcpyHostToDevice, s));
  if (C) CK(cudaMemcpyAsync(d_cust, cust, sizeof(int) * C, cudaMemcpyHostToDevice, s));
  if (R) {
    CK(cudaMemcpyAsync(d_dep, dep, sizeof(int) * R, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_arr, arr, sizeof(int) * R, cudaMemcpyHostToDevice, s));
  }
  CK(cudaMemcpyAsync(p->P.lam, lam, sizeof(double) * 4 * B, cudaMemcpyHostToDevice, s));
  p->B = B;
  if (B > 0) {
    launch_unpack(I, p->P, B, d_rbase, d_coff, d_cust, d_dep, d_arr, s);
    launch_rebuild(I, p->P, B, I.win, s);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  return MDR_OK;
}

static int download_impl(mdr_pop *p, int best, int32_t *rbase, int32_t *coff, int32_t *cust, int32_t *dep,
                         int32_t *arr, int32_t *n_routes, int32_t *n_cust, cudaStream_t s, int b0 = 0, int nb = -1) {
  int B = nb < 0 ? p->B : nb;
  int cap_r = *n_routes, cap_c = *n_cust;
  size_t need = (size_t)(B + 1) + (cap_r + 1) + cap_c + 2 * (size_t)cap_r;
  int rc = ensure_xfer(p, need);
  if (rc) return rc;
  int *d_rbase = p->d_xfer, *d_coff = d_rbase + B + 1, *d_cust = d_coff + cap_r + 1, *d_dep = d_cust + cap_c,
      *d_arr = d_dep + cap_r;
  launch_pack(p->P, b0, B, best, d_rbase, d_coff, d_cust, d_dep, d_arr, p->d_hdr, cap_r, cap_c, s);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(p->h_hdr, p->d_hdr, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  int R = p->h_hdr[0], C = p->h_hdr[1];
  *n_routes = R;
  *n_cust = C;
  if (R > cap_r || C > cap_c) return fail(MDR_ERR_CAPACITY, "download buffers too small");
  CK(cudaMemcpyAsync(rbase, d_rbase, sizeof(int) * (B + 1), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(coff, d_coff, sizeof(int) * (R + 1), cudaMemcpyDeviceToHost, s));
  if (C) CK(cudaMemcpyAsync(cust, d_cust, sizeof(int) * C, cudaMemcpyDeviceToHost, s));
  if (R) {
    CK(cudaMemcpyAsync(dep, d_dep, sizeof(int) * R, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(arr, d_arr, sizeof(int) * R, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  if (R == 0) coff[0] = 0;
  return MDR_OK;
}

int mdr_pop_download(mdr_pop *p, int32_t *rbase, int32_t *coff, int32_t *cust, int32_t *dep, int32_t *arr,
                     double *lam, int32_t *n_routes, int32_t *n_cust, void *stream) {
  if (!p) return fail(MDR_ERR_ARG, "null pop");
  CK(cudaSetDevice(p->inst->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = download_impl(p, 0, rbase, coff, cust, dep, arr, n_routes, n_cust, s);
  if (rc) return rc;
  if (lam) {
    CK(cudaMemcpyAsync(lam, p->P.lam, sizeof(double) * 4 * p->B, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return MDR_OK;
}

int mdr_pop_download_range(mdr_pop *p, int32_t b0, int32_t nb, int32_t *rbase, int32_t *coff, int32_t *cust,
                           int32_t *dep, int32_t *arr, int32_t *n_routes, int32_t *n_cust, void *stream) {
  if (!p || b0 < 0 || nb < 0 || b0 + nb > p->B) return fail(MDR_ERR_ARG, "individual range out of bounds");
  CK(cudaSetDevice(p->inst->device));
  return download_impl(p, 0, rbase, coff, cust, dep, arr, n_routes, n_cust, (cudaStream_t)stream, b0, nb);
}

int mdr_pop_download_best(mdr_pop *p, int32_t *rbase, int32_t *coff, int32_t *cust, int32_t *dep, int32_t *arr,
                          double *bestD, int32_t *n_routes, int32_t *n_cust, void *stream) {
  if (!p) return fail(MDR_ERR_ARG, "null pop");
  CK(cudaSetDevice(p->inst->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = download_impl(p, 1, rbase, coff, cust, dep, arr, n_routes, n_cust, s);
  if (rc) return rc;
  if (bestD) {
    std::vector<LsState> st(p->B);
    CK(cudaMemcpy(st.data(), p->P.st, sizeof(LsState) * p->B, cudaMemcpyDeviceToHost));
    for (int b = 0; b < p->B; b++) bestD[b] = st[b].bestD;
  }
  return MDR_OK;
}

// ---------------------------------------------------------------------------
// operator-level API
// ---------------------------------------------------------------------------
struct NonZero {
  __host__ __device__ bool operator()(const unsigned long long &k) const { return k != 0ull; }
};

static int enumerate_keys(mdr_pop *p, int b, int op, unsigned long long **d_out, long long *n_out,
                          std::vector<void *> &tmp, cudaStream_t s) {
  const DevInst &I = p->inst->I;
  int m = 0;
  CK(cudaMemcpy(&m, p->P.m + b, sizeof(int), cudaMemcpyDeviceToHost));
  long long items = op_items(op, m, I.NC, I.W, I.ND, I.win, I.open, p->P.K);
  unsigned long long *keys = nullptr, *outk = nullptr;
  int *nsel = nullptr;
  DA(tmp, keys, items);
  DA(tmp, outk, items);
  DA(tmp, nsel, 1);
  launch_emit(I, p->P, b, op, items, keys, s);
  CK(cudaGetLastError());
  size_t tb = 0;
  CK(cub::DeviceSelect::If(nullptr, tb, keys, outk, nsel, (int)items, NonZero(), s));
  char *tst = nullptr;
  DA(tmp, tst, tb + 1);
  CK(cub::DeviceSelect::If(tst, tb, keys, outk, nsel, (int)items, NonZero(), s));
  int n = 0;
  if (items) CK(cudaMemcpyAsync(&n, nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *d_out = outk;
  *n_out = n;
  return MDR_OK;
}

static void free_all(std::vector<void *> &v) {
  for (void *q : v) cudaFree(q);
  v.clear();
}

int64_t mdr_count(mdr_pop *p, int32_t b, int32_t op) {
  if (!p || b < 0 || b >= p->B || op < 0 || op > 5) {
    fail(MDR_ERR_ARG, "bad individual or operator");
    return -1;
  }
  if (cudaSetDevice(p->inst->device) != cudaSuccess) return -1;
  std::vector<void *> tmp;
  unsigned long long *k;
  long long n;
  int rc = enumerate_keys(p, b, op, &k, &n, tmp, 0);
  free_all(tmp);
  return rc ? -1 : n;
}

int mdr_enumerate(mdr_pop *p, int32_t b, int32_t op, mdr_cands *out) {
  if (!p || !out || b < 0 || b >= p->B) return fail(MDR_ERR_ARG, "bad individual");
  if (op < 0 || op > 5) return fail(MDR_ERR_ARG, "unknown operator");
  CK(cudaSetDevice(p->inst->device));
  std::vector<void *> tmp;
  unsigned long long *dk;
  long long n;
  int rc = enumerate_keys(p, b, op, &dk, &n, tmp, 0);
  if (rc) { free_all(tmp); return rc; }
  if (n > out->n) {
    out->n = n;
    free_all(tmp);
    return fail(MDR_ERR_CAPACITY, "candidate buffers too small");
  }
  std::vector<unsigned long long> hk(n);
  if (n) cudaMemcpy(hk.data(), dk, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  free_all(tmp);
  for (long long i = 0; i < n; i++) {
    Cand c = unpack_key(hk[i]);
    out->r1[i] = c.r1; out->p1[i] = c.p1; out->r2[i] = c.r2; out->p2[i] = c.p2;
    out->len1[i] = c.l1; out->len2[i] = c.l2; out->rev1[i] = (uint8_t)c.rev1; out->rev2[i] = (uint8_t)c.rev2;
    out->depot[i] = c.depot; out->mode[i] = c.mode;
  }
  out->n = n;
  return MDR_OK;
}

static int upload_cands(const mdr_cands *cs, MatCands &mc, std::vector<void *> &tmp, cudaStream_t s) {
  long long n = cs->n;
  long long *f[8];
  const int64_t *src[8] = {cs->r1, cs->p1, cs->r2, cs->p2, cs->len1, cs->len2, cs->depot, cs->mode};
  for (int i = 0; i < 8; i++) {
    DA(tmp, f[i], n);
    if (n) CK(cudaMemcpyAsync(f[i], src[i], n * sizeof(long long), cudaMemcpyHostToDevice, s));
  }
  unsigned char *r1 = nullptr, *r2 = nullptr;
  DA(tmp, r1, n);
  DA(tmp, r2, n);
  if (n) {
    CK(cudaMemcpyAsync(r1, cs->rev1, n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(r2, cs->rev2, n, cudaMemcpyHostToDevice, s));
  }
  mc.r1 = f[0]; mc.p1 = f[1]; mc.r2 = f[2]; mc.p2 = f[3]; mc.len1 = f[4]; mc.len2 = f[5]; mc.depot = f[6];
  mc.mode = f[7]; mc.rev1 = r1; mc.rev2 = r2; mc.n = n;
  return MDR_OK;
}

static int check_cands(mdr_pop *p, int b, int op, const mdr_cands *cs) {
  int m = 0;
  CK(cudaMemcpy(&m, p->P.m + b, sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int4> meta(m > 0 ? m : 1);
  if (m) CK(cudaMemcpy(meta.data(), p->P.rmeta + (size_t)b * p->P.J, sizeof(int4) * m, cudaMemcpyDeviceToHost));
  const DevInst &I = p->inst->I;
  for (long long i = 0; i < cs->n; i++) {
    long long r1 = cs->r1[i], r2 = cs->r2[i];
    bool two = (op == 0 || op == 1) ? r1 != r2 : op == 2;
    if (r1 < 0 || r1 >= m) return fail(MDR_ERR_ARG, "candidate r1 out of range");
    if ((two || op == 0 || op == 1) && (r2 < 0 || r2 >= m)) return fail(MDR_ERR_ARG, "candidate r2 out of range");
    long long k1 = meta[r1].x;
    long long p1 = cs->p1[i], p2 = cs->p2[i], l1 = cs->len1[i], l2 = cs->len2[i];
    if (p1 < 0 || p1 > k1 || l1 < 0 || l1 > 2 || l2 < 0 || l2 > 2) return fail(MDR_ERR_ARG, "candidate position out of range");
    if ((op == 0 || op == 1) && p1 + l1 > k1) return fail(MDR_ERR_ARG, "segment exceeds route");
    if (op == 0 || op == 1 || op == 2) {
      long long k2 = meta[r2].x;
      if (p2 < 0 || p2 > k2) return fail(MDR_ERR_ARG, "candidate p2 out of range");
      if (op == 1 && p2 + l2 > k2) return fail(MDR_ERR_ARG, "segment exceeds route");
    }
    if (op == 3 && (p2 < p1 || p2 >= k1)) return fail(MDR_ERR_ARG, "2-opt positions out of range");
    if (op == 4 && (p1 >= k1 || cs->depot[i] < 0 || cs->depot[i] >= I.ND)) return fail(MDR_ERR_ARG, "depot-insert out of range");
    if (op == 5 && (cs->depot[i] < 0 || cs->depot[i] >= I.ND || cs->mode[i] < 0 || cs->mode[i] > 2))
      return fail(MDR_ERR_ARG, "depot-replace out of range");
  }
  return MDR_OK;
}

int mdr_evaluate(mdr_pop *p, int32_t b, int32_t op, const mdr_cands *cs, const double lam[4], mdr_deltas *out) {
  if (!p || !cs || !out || b < 0 || b >= p->B) return fail(MDR_ERR_ARG, "bad individual");
  if (op < 0 || op > 5) return fail(MDR_ERR_ARG, "unknown operator");
  CK(cudaSetDevice(p->inst->device));
  int rc = check_cands(p, b, op, cs);
  if (rc) return rc;
  cudaStream_t s = 0;
  std::vector<void *> tmp;
  MatCands mc;
  rc = upload_cands(cs, mc, tmp, s);
  if (rc) { free_all(tmp); return rc; }
  long long n = cs->n;
  double *dl = nullptr, *dd = nullptr;
  unsigned char *fn = nullptr;
  if ((rc = dalloc(tmp, &dl, 4)) || (rc = dalloc(tmp, &dd, 6 * n)) || (rc = dalloc(tmp, &fn, n))) {
    free_all(tmp);
    return rc;
  }
  cudaMemcpyAsync(dl, lam, 4 * sizeof(double), cudaMemcpyHostToDevice, s);
  MatDeltas md{dd, dd + n, dd + 2 * n, dd + 3 * n, dd + 4 * n, dd + 5 * n, fn};
  launch_eval_mat(p->inst->I, p->P, b, op, mc, dl, md, p->inst->I.win, s);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { free_all(tmp); return fail(MDR_ERR_CUDA, cudaGetErrorString(e)); }
  double *hs[6] = {out->dD, out->dV1, out->dV2, out->dV3, out->dV4, out->dF};
  for (int f = 0; f < 6; f++)
    if (n) cudaMemcpy(hs[f], dd + f * n, n * sizeof(double), cudaMemcpyDeviceToHost);
  if (n) cudaMemcpy(out->fleet_neutral, fn, n, cudaMemcpyDeviceToHost);
  free_all(tmp);
  return MDR_OK;
}

struct OKI {
  unsigned long long o, k;
  long long i;
};
struct OKIMin {
  __host__ __device__ OKI operator()(const OKI &a, const OKI &b) const {
    if (a.o != b.o) return a.o < b.o ? a : b;
    if (a.k != b.k) return a.k < b.k ? a : b;
    return a.i <= b.i ? a : b;
  }
};
struct MakeOKI {
  const unsigned long long *o, *k;
  __host__ __device__ OKI operator()(long long i) const { return OKI{o[i], k[i], i}; }
};

__global__ void k_gather_u64(const unsigned long long *src, const long long *idx, unsigned long long *dst, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

int mdr_leader_followers(mdr_pop *p, const mdr_cands *cs, const mdr_deltas *d, int32_t multi_move, int64_t *leader,
                         int64_t *followers, int64_t *n_followers) {
  if (!p || !cs || !d || !leader) return fail(MDR_ERR_ARG, "null argument");
  CK(cudaSetDevice(p->inst->device));
  *leader = -1;
  if (n_followers) *n_followers = 0;
  long long n = cs->n;
  if (n == 0) return MDR_OK;
  for (long long i = 0; i < n; i++) {
    if (cs->r1[i] < -1 || cs->r1[i] > 4093 || cs->r2[i] < -1 || cs->r2[i] > 4093 || cs->p1[i] < -1 ||
        cs->p1[i] > 510 || cs->p2[i] < -1 || cs->p2[i] > 510 || cs->len1[i] < 0 || cs->len1[i] > 3 ||
        cs->len2[i] < 0 || cs->len2[i] > 3 || cs->depot[i] < -1 || cs->depot[i] > 254 || cs->mode[i] < -1 ||
        cs->mode[i] > 2)
      return fail(MDR_ERR_ARG, "candidate field outside the packed-key range");
  }
  cudaStream_t s = 0;
  std::vector<void *> tmp;
  MatCands mc;
  int rc = upload_cands(cs, mc, tmp, s);
  if (rc) { free_all(tmp); return rc; }
  double *dd = nullptr;
  unsigned char *fn = nullptr, *flag = nullptr;
  unsigned long long *ord = nullptr, *key = nullptr;
  int *nan = nullptr;
#define TA(ptr, cnt) if ((rc = dalloc(tmp, &(ptr), (cnt)))) { free_all(tmp); return rc; }
  TA(dd, 6 * n);
  TA(fn, n);
  TA(flag, n);
  TA(ord, n);
  TA(key, n);
  TA(nan, 1);
  const double *hs[6] = {d->dD, d->dV1, d->dV2, d->dV3, d->dV4, d->dF};
  for (int f = 0; f < 6; f++) cudaMemcpyAsync(dd + f * n, hs[f], n * sizeof(double), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(fn, d->fleet_neutral, n, cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(nan, 0, sizeof(int), s);
  MatDeltas md{dd, dd + n, dd + 2 * n, dd + 3 * n, dd + 4 * n, dd + 5 * n, fn};
  launch_lf_prep(mc, md, ord, key, flag, nan, s);
  // leader: min (ord(dF), key, index)  (batch.py:587-597, lexsort tie-break)
  OKI *dmin = nullptr;
  TA(dmin, 1);
  cub::CountingInputIterator<long long> cnt(0);
  cub::TransformInputIterator<OKI, MakeOKI, cub::CountingInputIterator<long long>> it(cnt, MakeOKI{ord, key});
  size_t tb = 0;
  OKI init{~0ull, ~0ull, (long long)n};
  CK(cub::DeviceReduce::Reduce(nullptr, tb, it, dmin, (int)n, OKIMin(), init, s));
  char *tst = nullptr;
  TA(tst, tb + 1);
  CK(cub::DeviceReduce::Reduce(tst, tb, it, dmin, (int)n, OKIMin(), init, s));
  OKI hmin;
  int hnan = 0;
  cudaMemcpyAsync(&hmin, dmin, sizeof(OKI), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&hnan, nan, sizeof(int), cudaMemcpyDeviceToHost, s);
  CK(cudaStreamSynchronize(s));
  auto unord_h = [](unsigned long long o) {
    unsigned long long u = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
    double x;
    memcpy(&x, &u, 8);
    return x;
  };
  if (hnan || hmin.o == ~0ull || !(unord_h(hmin.o) < -MDR_EPS)) {
    free_all(tmp);
    return MDR_OK;
  }
  *leader = hmin.i;
  if (multi_move && followers && n_followers) {
    // followers: flagged, minus the leader index, sorted by (dF, key, index) (batch.py:600-613)
    cudaMemsetAsync(flag + hmin.i, 0, 1, s);
    long long *fidx = nullptr, *fidx2 = nullptr;
    int *nsel = nullptr;
    unsigned long long *k1 = nullptr, *k2 = nullptr;
    TA(fidx, n);
    TA(fidx2, n);
    TA(nsel, 1);
    TA(k1, n);
    TA(k2, n);
    size_t t2 = 0;
    CK(cub::DeviceSelect::Flagged(nullptr, t2, cnt, flag, fidx, nsel, (int)n, s));
    char *ts2 = nullptr;
    TA(ts2, t2 + 1);
    CK(cub::DeviceSelect::Flagged(ts2, t2, cnt, flag, fidx, nsel, (int)n, s));
    int nf = 0;
    cudaMemcpyAsync(&nf, nsel, sizeof(int), cudaMemcpyDeviceToHost, s);
    CK(cudaStreamSynchronize(s));
    if (nf > 0) {
      int gb = (nf + 255) / 256;
      // stable LSD: sort by key, then by ord(dF)
      k_gather_u64<<<gb, 256, 0, s>>>(key, fidx, k1, nf);
      size_t t3 = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, t3, k1, k2, fidx, fidx2, nf, 0, 64, s));
      char *ts3 = nullptr;
      TA(ts3, t3 + 1);
      CK(cub::DeviceRadixSort::SortPairs(ts3, t3, k1, k2, fidx, fidx2, nf, 0, 58, s));
      k_gather_u64<<<gb, 256, 0, s>>>(ord, fidx2, k1, nf);
      CK(cub::DeviceRadixSort::SortPairs(ts3, t3, k1, k2, fidx2, fidx, nf, 0, 64, s));
      CK(cudaMemcpyAsync(followers, fidx, sizeof(long long) * nf, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    *n_followers = nf;
  }
#undef TA
  free_all(tmp);
  return MDR_OK;
}

int mdr_totals(mdr_pop *p, int32_t b, double out[5]) {
  if (!p || b < 0 || b >= p->B) return fail(MDR_ERR_ARG, "bad individual");
  CK(cudaSetDevice(p->inst->device));
  double *d = nullptr;
  CK(cudaMalloc(&d, 5 * sizeof(double)));
  launch_totals(p->inst->I, p->P, b, d, 0);
  cudaError_t e = cudaMemcpy(out, d, 5 * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(MDR_ERR_CUDA, cudaGetErrorString(e));
  return MDR_OK;
}

// ---------------------------------------------------------------------------
// population-batched local search
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// operator permutation stream: CPython's random.Random.shuffle on MT19937
// (Modules/_randommodule.c genrand_uint32, Lib/random.py shuffle /
// _randbelow_with_getrandbits), driven by the state rng.getstate() exposes
// ---------------------------------------------------------------------------
static uint32_t mt_next(uint32_t *mt, uint32_t *idx) {
  const int N = 624, M = 397;
  const uint32_t A = 0x9908b0dfU, UP = 0x80000000U, LO = 0x7fffffffU;
  uint32_t y;
  if (*idx >= (uint32_t)N) {
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
    *idx = 0;
  }
  y = mt[(*idx)++];
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680U;
  y ^= (y << 15) & 0xefc60000U;
  y ^= (y >> 18);
  return y;
}

int mdr_shuffle_stream(uint32_t *state, int32_t n_items, const uint8_t *items, int32_t n_passes, uint8_t *out) {
  if (!state || !items || n_items < 1 || n_items > 64 || n_passes < 0) return fail(MDR_ERR_ARG, "bad shuffle arguments");
  uint32_t *mt = state, *idx = state + 624;
  if (*idx > 624) return fail(MDR_ERR_ARG, "bad MT19937 state index");
  uint8_t tmp[64];
  for (int p = 0; p < n_passes; p++) {
    for (int i = 0; i < n_items; i++) tmp[i] = items[i];
    for (int i = n_items - 1; i >= 1; i--) {
      uint32_t n = (uint32_t)i + 1, k = 0;
      while ((1u << k) <= n && k < 32) k++;  // n.bit_length()
      uint32_t r;
      do { r = mt_next(mt, idx) >> (32 - k); } while (r >= n);
      uint8_t t = tmp[i];
      tmp[i] = tmp[r];
      tmp[r] = t;
    }
    if (out)
      for (int i = 0; i < n_items; i++) out[(size_t)p * n_items + i] = tmp[i];
  }
  return MDR_OK;
}

int mdr_repair(mdr_pop *p, int32_t op, const int32_t *pend_off, const int32_t *pend, mdr_repair_stats *stats,
               void *stream) {
  if (!p || !pend_off || (pend_off[p->B] > 0 && !pend)) return fail(MDR_ERR_ARG, "null argument");
  if (op < 0 || op > 3) return fail(MDR_ERR_ARG, "op must be FBI(0), IBI(1), FRI(2) or IRI(3)");
  const int B = p->B;
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(p->inst->device));
  const DevInst &I = p->inst->I;
  DevPop &P = p->P;
  // pending lists sorted ascending (repair_insert sorts, genetic.py:198); duplicates rejected
  std::vector<int> off(B + 1, 0), srt;
  int Pmax = 0;
  for (int b = 0; b < B; b++) {
    const int n = pend_off[b + 1] - pend_off[b];
    if (n < 0) return fail(MDR_ERR_ARG, "pend_off must be non-decreasing");
    std::vector<int> v(pend + pend_off[b], pend + pend_off[b + 1]);
    std::sort(v.begin(), v.end());
    for (int i = 0; i < n; i++) {
      if (v[i] < I.ND || v[i] >= I.N) return fail(MDR_ERR_ARG, "pending node is not a customer");
      if (i && v[i] == v[i - 1]) return fail(MDR_ERR_ARG, "pending customer listed twice");
    }
    srt.insert(srt.end(), v.begin(), v.end());
    off[b + 1] = off[b] + n;
    Pmax = std::max(Pmax, n);
  }
  if (Pmax > 4096) return fail(MDR_ERR_ARG, "more than 4096 pending customers in one individual");
  const size_t tab = (size_t)P.Bcap * P.J * P.Kp * repair_attr_bytes();  // bytes
  const size_t cache = (size_t)std::max(B, 1) * std::max(Pmax, 1) * P.J;
  const size_t pn = (size_t)(B + 1) + srt.size() + 1, nb = (size_t)std::max(B, 1);
  int rc;
  if ((rc = regrow(&p->rp_pre, p->rp_cap[0], tab)) || (rc = regrow(&p->rp_suf, p->rp_cap[1], tab)) ||
      (rc = regrow(&p->rp_c1, p->rp_cap[2], cache)) || (rc = regrow(&p->rp_c2, p->rp_cap[3], cache)) ||
      (rc = regrow(&p->rp_p1, p->rp_cap[4], cache)) || (rc = regrow(&p->rp_pend, p->rp_cap[5], pn)) ||
      (rc = regrow(&p->rp_status, p->rp_cap[6], nb)) || (rc = regrow(&p->rp_stats, p->rp_cap[7], 3 * nb)) ||
      (rc = regrow(&p->rp_fold, p->rp_cap[8], nb * std::max(Pmax, 1) * 2)) ||
      (rc = regrow(&p->rp_foldi, p->rp_cap[9], nb * std::max(Pmax, 1) * 3)))
    return rc;
  int *d_off = p->rp_pend, *d_pend = p->rp_pend + B + 1;
  CK(cudaMemcpyAsync(d_off, off.data(), sizeof(int) * (B + 1), cudaMemcpyHostToDevice, s));
  if (!srt.empty()) CK(cudaMemcpyAsync(d_pend, srt.data(), sizeof(int) * srt.size(), cudaMemcpyHostToDevice, s));
  launch_repair(I, P, B, op, d_off, d_pend, p->rp_pre, p->rp_suf, p->rp_c1, p->rp_c2, p->rp_p1, p->rp_fold,
                p->rp_foldi, std::max(Pmax, 1), p->rp_status, p->rp_stats, s);
  CK(cudaGetLastError());
  std::vector<int> st(std::max(B, 1));
  std::vector<long long> ev((size_t)std::max(B, 1) * 3);
  if (B) {
    CK(cudaMemcpyAsync(st.data(), p->rp_status, sizeof(int) * B, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ev.data(), p->rp_stats, sizeof(long long) * 3 * B, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  int worst = MDR_OK;
  for (int b = 0; b < B; b++) {
    if (stats) {
      stats[b].status = st[b];
      stats[b].inserted = off[b + 1] - off[b];
      stats[b].slot_evals = ev[3 * b];
      stats[b].ref_slot_evals = ev[3 * b + 1];
      stats[b].need_j = (int)(ev[3 * b + 2] >> 32);
      stats[b].need_k = (int)(ev[3 * b + 2] & 0xffffffff);
    }
    if (st[b] && !worst) worst = st[b];
  }
  if (worst == MDR_ERR_ARG) return fail(MDR_ERR_ARG, "pending customer is already routed");
  if (worst == MDR_ERR_CAPACITY) return fail(MDR_ERR_CAPACITY, "repair needs more routes (J) or a longer route (K)");
  if (worst) return fail(worst, "repair failed");
  // the population is left ready for mdr_local_search / mdr_pop_download
  if (B > 0) launch_rebuild(I, P, B, I.win, s);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  return MDR_OK;
}

int mdr_construct(mdr_pop *p, int32_t B, const int32_t *ooff, const int32_t *order, int32_t *n_left, int32_t *left,
                  void *stream) {
  if (!p || !ooff || !n_left || !left) return fail(MDR_ERR_ARG, "null argument");
  const DevInst &I = p->inst->I;
  DevPop &P = p->P;
  if (B < 0 || B > P.Bcap) return fail(MDR_ERR_ARG, "B exceeds the population capacity");
  const int NC = I.N - I.ND;
  const int tot = ooff[(size_t)B * I.ND];
  if (tot > 0 && !order) return fail(MDR_ERR_ARG, "null order");
  int Jd = 1;
  for (int b = 0; b < B; b++) {
    std::vector<char> seen(I.N, 0);
    for (int d = 0; d < I.ND; d++) {
      const int a = ooff[b * I.ND + d], e = ooff[b * I.ND + d + 1];
      if (e < a) return fail(MDR_ERR_ARG, "ooff must be non-decreasing");
      Jd = std::max(Jd, e - a);
      for (int t = a; t < e; t++) {
        const int c = order[t];
        if (c < I.ND || c >= I.N || seen[c]) return fail(MDR_ERR_ARG, "order holds a non-customer or a repeat");
        seen[c] = 1;
      }
    }
  }
  Jd = std::min(Jd, P.J);
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(p->inst->device));
  const size_t tab = (size_t)std::max(B, 1) * Jd * P.Kp * repair_attr_bytes();
  int rc;
  if ((rc = regrow(&p->rp_pre, p->rp_cap[0], tab)) || (rc = regrow(&p->rp_suf, p->rp_cap[1], tab))) return rc;
  int *d_buf = nullptr;
  const size_t nbuf = (size_t)B * I.ND + 1 + tot + 2 * (size_t)std::max(B, 1) + (size_t)std::max(B, 1) * NC;
  CK(cudaMalloc(&d_buf, sizeof(int) * nbuf));
  int *d_ooff = d_buf, *d_order = d_ooff + (size_t)B * I.ND + 1, *d_nl = d_order + tot, *d_st = d_nl + std::max(B, 1),
      *d_left = d_st + std::max(B, 1);
  std::vector<int> st(std::max(B, 1));
  auto run = [&]() -> int {
    CK(cudaMemcpyAsync(d_ooff, ooff, sizeof(int) * ((size_t)B * I.ND + 1), cudaMemcpyHostToDevice, s));
    if (tot) CK(cudaMemcpyAsync(d_order, order, sizeof(int) * tot, cudaMemcpyHostToDevice, s));
    launch_construct(I, P, B, d_ooff, d_order, p->rp_pre, p->rp_suf, Jd, d_nl, d_left, d_st, s);
    CK(cudaGetLastError());
    if (B) {
      CK(cudaMemcpyAsync(st.data(), d_st, sizeof(int) * B, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(n_left, d_nl, sizeof(int) * B, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(left, d_left, sizeof(int) * (size_t)B * NC, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    return MDR_OK;
  };
  rc = run();
  cudaFree(d_buf);
  if (rc) return rc;
  for (int b = 0; b < B; b++)
    if (st[b]) return fail(MDR_ERR_CAPACITY, "construction needs more routes (J) or a longer route (K)");
  p->B = B;
  if (B > 0) launch_rebuild(I, P, B, I.win, s);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  return MDR_OK;
}

int mdr_pop_breakdown(mdr_pop *p, const double *lam, double *out, void *stream) {
  if (!p || !out) return fail(MDR_ERR_ARG, "null argument");
  const int B = p->B;
  if (B == 0) return MDR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(p->inst->device));
  int rc;
  if ((rc = regrow(&p->bd_rt, p->rp_cap[10], (size_t)B * p->P.J * 5)) ||
      (rc = regrow(&p->bd_io, p->rp_cap[11], (size_t)B * 10)))
    return rc;
  double *d_lam = p->bd_io, *d_out = p->bd_io + 4 * (size_t)B;
  if (lam) CK(cudaMemcpyAsync(d_lam, lam, sizeof(double) * 4 * B, cudaMemcpyHostToDevice, s));
  else CK(cudaMemcpyAsync(d_lam, p->P.lam, sizeof(double) * 4 * B, cudaMemcpyDeviceToDevice, s));
  launch_breakdown(p->inst->I, p->P, B, d_lam, p->bd_rt, d_out, s);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d_out, sizeof(double) * 6 * B, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return MDR_OK;
}

int mdr_pop_info(mdr_pop *p, int32_t out[4]) {
  if (!p || !out) return fail(MDR_ERR_ARG, "null argument");
  out[0] = p->P.staged;
  out[1] = p->P.ct;
  out[2] = p->P.ct == MDR_LARGE_CT ? MDR_LARGE_CU : MDR_SMALL_CU;
  out[3] = p->P.Bcap;
  return MDR_OK;
}

int mdr_set_profiling(mdr_pop *p, int32_t on) {
  if (!p) return fail(MDR_ERR_ARG, "null pop");
  p->profiling = on;
  return MDR_OK;
}

int mdr_get_timing(mdr_pop *p, mdr_timing *out) {
  if (!p || !out) return fail(MDR_ERR_ARG, "null argument");
  *out = p->tm;
  return MDR_OK;
}

int mdr_local_search(mdr_pop *p, const mdr_ls_cfg *cfg, mdr_ls_stats *stats, void *stream) {
  if (!p || !cfg) return fail(MDR_ERR_ARG, "null argument");
  if (cfg->depth < 1) return fail(MDR_ERR_ARG, "depth must be >= 1");
  if (!(cfg->kappa > 0.0 && cfg->kappa < 1.0)) return fail(MDR_ERR_ARG, "kappa must lie in (0, 1)");
  if (cfg->n_ops < 1 || cfg->n_ops > 6 || cfg->max_passes < 1 || !cfg->perms)
    return fail(MDR_ERR_ARG, "bad operator permutation stream");
  const int B = p->B;
  CK(cudaSetDevice(p->inst->device));
  cudaStream_t s = (cudaStream_t)stream;
  const DevInst &I = p->inst->I;
  size_t np = (size_t)B * cfg->max_passes * cfg->n_ops;
  for (size_t i = 0; i < np; i++)
    if (cfg->perms[i] > 5 || (I.win && cfg->perms[i] == 3)) return fail(MDR_ERR_ARG, "bad operator in permutation");
  if (np > p->perms_cap) {
    if (p->d_perms) cudaFree(p->d_perms);
    p->d_perms = nullptr;
    CK(cudaMalloc(&p->d_perms, np + 1));
    p->perms_cap = np;
  }
  if (np) CK(cudaMemcpyAsync(p->d_perms, cfg->perms, np, cudaMemcpyHostToDevice, s));
  DevPop P = p->P;
  P.perms = p->d_perms;
  P.maxp = cfg->max_passes;
  P.nops = cfg->n_ops;
  std::vector<LsState> st0(B > 0 ? B : 1);
  for (int b = 0; b < B; b++) {
    memset(&st0[b], 0, sizeof(LsState));
    st0[b].bestD = INFINITY;
  }
  if (B) {
    CK(cudaMemcpyAsync(P.st, st0.data(), sizeof(LsState) * B, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(P.cands, 0, sizeof(unsigned long long) * B * 6, s));
    CK(cudaMemsetAsync(P.best_m, 0, sizeof(int) * B, s));
  }
  LsParams L;
  memset(&L, 0, sizeof(L));  // padding too: the bytes key the cached round graph
  L.depth = cfg->depth;
  L.multi_move = cfg->multi_move ? 1 : 0;
  L.kappa = cfg->kappa;
  L.lam_min = cfg->lam_min;
  L.lam_max = cfg->lam_max;
  L.B = B;
  L.snapshot = cfg->snapshot_best ? 1 : 0;
  L.trace = cfg->trace ? 1 : 0;
  P.trace = nullptr;
  P.trcount = nullptr;
  P.tcap = 0;
  if (L.trace && B) {  // a step selects at most one move per route: depth * (2 + J) words bound it
    const long long per = (long long)cfg->depth * (2 + P.J);
    int rc;
    if ((rc = regrow(&p->tr_buf, p->tr_cap[0], (size_t)B * per)) || (rc = regrow(&p->tr_cnt, p->tr_cap[1], (size_t)B)))
      return rc;
    CK(cudaMemsetAsync(p->tr_cnt, 0, sizeof(long long) * B, s));
    P.trace = p->tr_buf;
    P.trcount = p->tr_cnt;
    P.tcap = per;
    p->tr_per = per;
  }
  static const int rps_env = getenv("MDR_RPS") ? atoi(getenv("MDR_RPS")) : 0;  // A/B override
  // 16 rounds per host poll: with the graph kept across calls, +0.1-0.3 % over 8 at C2-C4 (C1 -2.5 %)
  const int rps = rps_env > 0 ? rps_env : cfg->rounds_per_sync > 0 ? cfg->rounds_per_sync : 16;
  auto t0 = std::chrono::steady_clock::now();
  int prof = p->profiling;
  if (prof) CK(cudaEventRecord(p->ev[6], s));
  long long rounds = 0;
  long long ev_used = 0;
  const bool dbg = getenv("MDR_SYNC_DEBUG") != nullptr;  // sync + check after every kernel
  auto ev_at = [&](long long i) -> cudaEvent_t {
    while ((long long)p->rev.size() <= i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      p->rev.push_back(e);
    }
    return p->rev[i];
  };
  // the round loop runs on a private stream joined to the caller's; after a
  // first eager batch, each batch of rps rounds is one CUDA graph launch
  const bool graph = !prof && !dbg && !getenv("MDR_NO_GRAPH");
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cs = s;
  s = p->ls;
  CK(cudaEventRecord(p->join[0], cs));
  CK(cudaStreamWaitEvent(s, p->join[0], 0));
  long long batches = 0;
  while (B > 0) {
    if (graph && batches > 0) {
      if (!gexec) {
        // the captured kernels hold (I, P, L) by value: reuse the previous call's
        // graph when those bytes and the batch length are unchanged (instantiating
        // it costs ~0.1 ms per round; a short descent is a few ms)
        std::vector<unsigned char> key(sizeof(DevInst) + sizeof(DevPop) + sizeof(LsParams) + sizeof(int));
        unsigned char *kp = key.data();
        memcpy(kp, &I, sizeof(DevInst));
        memcpy(kp + sizeof(DevInst), &P, sizeof(DevPop));
        memcpy(kp + sizeof(DevInst) + sizeof(DevPop), &L, sizeof(LsParams));
        memcpy(kp + sizeof(DevInst) + sizeof(DevPop) + sizeof(LsParams), &rps, sizeof(int));
        if (p->gx && p->gkey == key) {
          gexec = p->gx;
        } else {
          if (p->gx) cudaGraphExecDestroy(p->gx);
          p->gx = nullptr;
          cudaGraph_t gr;
          CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
          for (int r = 0; r < rps; r++) {
            launch_plan(I, P, L, s);
            launch_eval(I, P, L, p->grid, I.win, s, p->side, p->fev);
            launch_eval_g(I, P, L, p->grid, I.win, s);
            launch_select(I, P, L, I.win, s);
          }
          CK(cudaStreamEndCapture(s, &gr));
          CK(cudaGraphInstantiate(&gexec, gr, 0));
          cudaGraphDestroy(gr);
          p->gx = gexec;
          p->gkey.swap(key);
        }
      }
      CK(cudaGraphLaunch(gexec, s));
      rounds += rps;
    } else
    for (int r = 0; r < rps; r++) {
      if (prof) cudaEventRecord(ev_at(ev_used), s);
      launch_plan(I, P, L, s);
      if (dbg && cudaStreamSynchronize(s)) return fail(MDR_ERR_CUDA, "k_plan failed");
      if (prof) cudaEventRecord(ev_at(ev_used + 1), s);
      cudaEvent_t *kt = nullptr;
      if (prof) {
        const size_t need = (size_t)(ev_used / 5 + 1) * 7;
        while (p->kev.size() < need) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          p->kev.push_back(e);
        }
        kt = p->kev.data() + (ev_used / 5) * 7;
      }
      launch_eval(I, P, L, p->grid, I.win, s, p->side, p->fev, kt);
      if (dbg && cudaStreamSynchronize(s)) return fail(MDR_ERR_CUDA, "k_eval failed");
      if (prof) cudaEventRecord(ev_at(ev_used + 2), s);
      launch_eval_g(I, P, L, p->grid, I.win, s);
      if (dbg && cudaStreamSynchronize(s)) return fail(MDR_ERR_CUDA, "k_eval_g failed");
      if (prof) cudaEventRecord(ev_at(ev_used + 3), s);
      launch_select(I, P, L, I.win, s);
      if (dbg && cudaStreamSynchronize(s)) return fail(MDR_ERR_CUDA, "k_select failed");
      if (prof) {
        cudaEventRecord(ev_at(ev_used + 4), s);
        ev_used += 5;
      }
      rounds++;
    }
    batches++;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(p->h_hdr, P.active, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (p->h_hdr[0] == 0) break;
    if (cfg->deadline_s >= 0) {
      double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > cfg->deadline_s) break;
    }
  }
  CK(cudaEventRecord(p->join[1], s));
  CK(cudaStreamWaitEvent(cs, p->join[1], 0));
  if (prof) {
    CK(cudaEventRecord(p->ev[7], s));
    CK(cudaEventSynchronize(p->ev[7]));
    float tot = 0;
    cudaEventElapsedTime(&tot, p->ev[6], p->ev[7]);
    p->tm.total_ms += tot;
    p->tm.rounds += rounds;
    FILE *rlog = getenv("MDR_ROUND_LOG") ? fopen(getenv("MDR_ROUND_LOG"), "w") : nullptr;
    for (long long e = 0; e + 4 < ev_used; e += 5) {
      float a = 0, b2 = 0, g = 0, c = 0;
      cudaEventElapsedTime(&a, p->rev[e], p->rev[e + 1]);
      cudaEventElapsedTime(&b2, p->rev[e + 1], p->rev[e + 2]);
      cudaEventElapsedTime(&g, p->rev[e + 2], p->rev[e + 3]);
      cudaEventElapsedTime(&c, p->rev[e + 3], p->rev[e + 4]);
      p->tm.plan_ms += a;
      p->tm.eval_ms += b2;
      p->tm.geval_ms += g;
      p->tm.select_ms += c;
      p->tm.eval_launches++;
      if (P.staged) {
        cudaEvent_t *kt = p->kev.data() + (e / 5) * 7;
        for (int q = 0; q < 6; q++) {
          float x = 0;
          cudaEventElapsedTime(&x, kt[q], kt[q + 1]);
          p->tm.kern_ms[q] += x;
        }
        p->tm.kern_rounds++;
      }
      if (rlog) fprintf(rlog, "%lld,%.4f,%.4f,%.4f,%.4f\n", e / 5, a, b2, g, c);
    }
    if (rlog) fclose(rlog);
  }
  if (!prof) p->tm.rounds += rounds;
  std::vector<LsState> st(B > 0 ? B : 1);
  std::vector<unsigned long long> cands((size_t)(B > 0 ? B : 1) * 6);
  if (B) {
    CK(cudaMemcpyAsync(st.data(), P.st, sizeof(LsState) * B, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(cands.data(), P.cands, sizeof(unsigned long long) * B * 6, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  int worst = MDR_OK;
  for (int b = 0; b < B; b++) {
    if (stats) {
      mdr_ls_stats &o = stats[b];
      o.passes = st[b].pass + 1;
      o.accepted = st[b].accepted;
      o.op_evals = st[b].op_evals;
      o.status = st[b].status;
      for (int q = 0; q < 6; q++) {
        o.cands[q] = (int64_t)cands[(size_t)b * 6 + q];
        if (prof) p->tm.cands_total += o.cands[q];
      }
      o.moves_applied = st[b].moves_applied;
      o.n_feasible = st[b].n_feasible;
      o.n_improving = st[b].n_improving;
      o.best_feasible_D = st[b].bestD;
      o.need_followers = st[b].need_f;
      o.need_queue = st[b].need_g;
      o.need_routes = st[b].need_j;
      o.need_positions = st[b].need_k;
    }
    if (st[b].status && !worst) worst = st[b].status;
  }
  if (worst == MDR_ERR_CAPACITY) return fail(worst, "capacity exceeded during local search (J_cap/K_cap/F_cap)");
  if (worst) return fail(worst, "local search stopped with an error status");
  return MDR_OK;
}

int mdr_pop_route_attrs(mdr_pop *p, int32_t b0, int32_t nb, double *out, void *stream) {
  if (!p || !out) return fail(MDR_ERR_ARG, "null argument");
  if (b0 < 0 || nb < 0 || b0 + nb > p->B) return fail(MDR_ERR_ARG, "individual range out of bounds");
  if (nb == 0) return MDR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(p->inst->device));
  const size_t n = (size_t)nb * p->P.J * 6;
  int rc;
  if ((rc = regrow(&p->ra_buf, p->ra_cap, n))) return rc;
  launch_route_attrs(p->inst->I, p->P, b0, nb, p->ra_buf, s);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, p->ra_buf, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return MDR_OK;
}

int mdr_pop_trace(mdr_pop *p, int32_t b, uint64_t *out, int64_t cap, int64_t *n) {
  if (!p || !n) return fail(MDR_ERR_ARG, "null argument");
  if (b < 0 || b >= p->B || !p->tr_buf || !p->tr_per) return fail(MDR_ERR_ARG, "no trace of this individual");
  CK(cudaSetDevice(p->inst->device));
  long long cnt = 0;
  CK(cudaMemcpy(&cnt, p->tr_cnt + b, sizeof(long long), cudaMemcpyDeviceToHost));
  *n = cnt;
  if (cnt > p->tr_per) return fail(MDR_ERR_CAPACITY, "trace overflow");
  if (!out || cap < cnt) return fail(MDR_ERR_CAPACITY, "trace output buffer too small");
  if (cnt) CK(cudaMemcpy(out, p->tr_buf + (size_t)b * p->tr_per, sizeof(uint64_t) * cnt, cudaMemcpyDeviceToHost));
  return MDR_OK;
}

int mdr_route_exchange(mdr_instance *inst, int32_t M, const int32_t *mroute, const int32_t *coff, const int32_t *cust,
                       const int32_t *dep, const int32_t *arr, int32_t B, const int32_t *main_idx,
                       const int32_t *donors, uint32_t *mt, const double *sigma_bounds, int32_t J_cap,
                       int32_t C_cap, int32_t *refs, int32_t *n_refs, int32_t *keep, int32_t *unrouted,
                       int32_t *n_unrouted, double *sigma) {
  if (!inst || M < 2 || B < 0 || !mroute || !coff || !dep || !arr || (B && (!main_idx || !donors || !mt ||
      !sigma_bounds || !refs || !n_refs || !keep || !unrouted || !n_unrouted || !sigma)))
    return fail(MDR_ERR_ARG, "bad argument");
  if (B == 0) return MDR_OK;
  const DevInst &I = inst->I;
  const int R = mroute[M], NC = I.N - I.ND, nc_all = coff[R];
  int jmax = 1;
  for (int m = 0; m < M; m++) {
    if (mroute[m + 1] < mroute[m]) return fail(MDR_ERR_ARG, "mroute must be non-decreasing");
    jmax = std::max(jmax, mroute[m + 1] - mroute[m]);
  }
  for (int b = 0; b < B; b++)
    if (main_idx[b] < 0 || main_idx[b] >= M) return fail(MDR_ERR_ARG, "main index out of range");
  for (size_t q = 0; q < (size_t)B * (M - 1); q++)
    if (donors[q] < 0 || donors[q] >= M) return fail(MDR_ERR_ARG, "donor index out of range");
  for (int q = 0; q < nc_all; q++)
    if (cust[q] < I.ND || cust[q] >= I.N) return fail(MDR_ERR_ARG, "route member is not a customer");
  CK(cudaSetDevice(inst->device));
  const int words = (I.N + 31) / 32;
  const int cnt_cap = std::max(I.N, J_cap * jmax + 3 * jmax);
  std::vector<void *> tmp;
  auto dmal = [&](size_t bytes) -> void * {
    void *q = nullptr;
    if (cudaMallocAsync(&q, bytes ? bytes : 1, 0) != cudaSuccess) return nullptr;  // pool: no device sync
    tmp.push_back(q);
    return q;
  };
  int rc = MDR_OK;
  auto run = [&]() -> int {
    XcPop X;
    XcJob Jb;
    XcOut O;
    int *d_pop = (int *)dmal(sizeof(int) * ((size_t)(M + 1) + (R + 1) + nc_all + 2 * (size_t)R));
    int *d_job = (int *)dmal(sizeof(int) * ((size_t)B + (size_t)B * (M - 1)));
    uint32_t *d_mt = (uint32_t *)dmal(sizeof(uint32_t) * 625 * (size_t)B);
    double *d_sig = (double *)dmal(sizeof(double) * 3 * (size_t)B);
    int *d_out = (int *)dmal(sizeof(int) * ((size_t)B * (2 * J_cap + C_cap + NC + 3)));
    int *d_scr = (int *)dmal(sizeof(int) * (size_t)B * (3 * (size_t)I.N + 3 * words + cnt_cap));
    long long *d_key = (long long *)dmal(sizeof(long long) * (size_t)B * cnt_cap);
    if (!d_pop || !d_job || !d_mt || !d_sig || !d_out || !d_scr || !d_key) return fail(MDR_ERR_CUDA, "cudaMalloc failed");
    int *p = d_pop;
    CK(cudaMemcpy(p, mroute, sizeof(int) * (M + 1), cudaMemcpyHostToDevice)); X.mroute = p; p += M + 1;
    CK(cudaMemcpy(p, coff, sizeof(int) * (R + 1), cudaMemcpyHostToDevice)); X.coff = p; p += R + 1;
    if (nc_all) CK(cudaMemcpy(p, cust, sizeof(int) * nc_all, cudaMemcpyHostToDevice));
    X.cust = p; p += nc_all;
    if (R) CK(cudaMemcpy(p, dep, sizeof(int) * R, cudaMemcpyHostToDevice));
    X.dep = p; p += R;
    if (R) CK(cudaMemcpy(p, arr, sizeof(int) * R, cudaMemcpyHostToDevice));
    X.arr = p;
    CK(cudaMemcpy(d_job, main_idx, sizeof(int) * B, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_job + B, donors, sizeof(int) * (size_t)B * (M - 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_mt, mt, sizeof(uint32_t) * 625 * (size_t)B, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_sig, sigma_bounds, sizeof(double) * 2 * (size_t)B, cudaMemcpyHostToDevice));
    Jb.main = d_job; Jb.donors = d_job + B; Jb.mt = d_mt; Jb.sig = d_sig;
    int *q = d_out;
    O.refs = q; q += (size_t)B * J_cap;
    O.orig = q; q += (size_t)B * J_cap;
    O.keep = q; q += (size_t)B * C_cap;
    O.unr = q; q += (size_t)B * NC;
    O.nref = q; q += B;
    O.nunr = q; q += B;
    O.status = q;
    O.sigma = d_sig + 2 * (size_t)B;
    O.Jcap = J_cap; O.Ccap = C_cap;
    int *sc = d_scr;
    int *prv = sc, *nxt = sc + (size_t)B * I.N, *own = sc + 2 * (size_t)B * I.N;
    unsigned *bits = (unsigned *)(sc + 3 * (size_t)B * I.N);
    int *cntp = (int *)(bits + (size_t)B * 3 * words);
    launch_exchange(I, X, Jb, O, B, M, prv, nxt, own, bits, cntp, d_key, cnt_cap, 0);
    CK(cudaGetLastError());
    std::vector<int> st(B);
    CK(cudaMemcpy(st.data(), O.status, sizeof(int) * B, cudaMemcpyDeviceToHost));
    for (int b = 0; b < B; b++)
      if (st[b]) return fail(st[b], "route exchange: capacity (J_cap / C_cap) exceeded");
    CK(cudaMemcpy(refs, O.refs, sizeof(int) * (size_t)B * J_cap, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(n_refs, O.nref, sizeof(int) * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(keep, O.keep, sizeof(int) * (size_t)B * C_cap, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(unrouted, O.unr, sizeof(int) * (size_t)B * NC, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(n_unrouted, O.nunr, sizeof(int) * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sigma, O.sigma, sizeof(double) * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(mt, d_mt, sizeof(uint32_t) * 625 * (size_t)B, cudaMemcpyDeviceToHost));
    return MDR_OK;
  };
  rc = run();
  for (void *t : tmp) cudaFreeAsync(t, 0);
  return rc;
}

int mdr_route_sim(mdr_instance *inst, int32_t n_routes, const int32_t *off, const int32_t *seq, int32_t want_min,
                  double *out) {
  if (!inst || n_routes < 0 || (n_routes > 0 && (!off || !seq || !out))) return fail(MDR_ERR_ARG, "null argument");
  if (n_routes == 0) return MDR_OK;
  const DevInst &I = inst->I;
  for (int r = 0; r < n_routes; r++) {
    if (off[r + 1] - off[r] < 1) return fail(MDR_ERR_ARG, "empty route sequence");
  }
  const int ns = off[n_routes];
  for (int i = 0; i < ns; i++)
    if (seq[i] < 0 || seq[i] >= I.N) return fail(MDR_ERR_ARG, "node id out of range");
  CK(cudaSetDevice(inst->device));
  int *d_off = nullptr, *d_seq = nullptr;
  double *d_raw = nullptr, *d_out = nullptr;
  int rc = MDR_OK;
  auto run = [&]() -> int {
    CK(cudaMallocAsync(&d_off, sizeof(int) * (n_routes + 1), 0));
    CK(cudaMallocAsync(&d_seq, sizeof(int) * ns, 0));
    CK(cudaMallocAsync(&d_raw, sizeof(double) * ns, 0));
    CK(cudaMallocAsync(&d_out, sizeof(double) * 6 * n_routes, 0));
    CK(cudaMemcpy(d_off, off, sizeof(int) * (n_routes + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_seq, seq, sizeof(int) * ns, cudaMemcpyHostToDevice));
    launch_route_sim(I, n_routes, d_off, d_seq, want_min, d_raw, d_out, 0);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, d_out, sizeof(double) * 6 * n_routes, cudaMemcpyDeviceToHost));
    return MDR_OK;
  };
  rc = run();
  if (d_off) cudaFreeAsync(d_off, 0);
  if (d_seq) cudaFreeAsync(d_seq, 0);
  if (d_raw) cudaFreeAsync(d_raw, 0);
  if (d_out) cudaFreeAsync(d_out, 0);
  return rc;
}

}  // extern "C"
