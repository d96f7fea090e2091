// mdr_kernels.cuh -- kernel launchers shared by mdr_api.cu
#pragma once
#include "mdr_device.cuh"

namespace mdr {

struct MatCands {  // device SoA of a materialised CandidateSet
  const long long *r1, *p1, *r2, *p2, *len1, *len2, *depot, *mode;
  const unsigned char *rev1, *rev2;
  long long n;
};

struct MatDeltas {
  double *dD, *dV1, *dV2, *dV3, *dV4, *dF;
  unsigned char *fn;
};

int mdr_fail(int code, const char *msg);  // sets mdr_last_error (mdr_api.cu)
void launch_rebuild(const DevInst &I, const DevPop &P, int B, bool win, cudaStream_t s);
void launch_repair(const DevInst &I, const DevPop &P, int B, int op, const int *pend_off, const int *pend,
                   void *pre, void *suf, double *c1, double *c2, int *p1, double *fold, int *foldi, int Pcap,
                   int *status, long long *stats, cudaStream_t s);
size_t repair_attr_bytes();
void launch_route_attrs(const DevInst &I, const DevPop &P, int b0, int nb, double *out, cudaStream_t s);
void launch_construct(const DevInst &I, const DevPop &P, int B, const int *ooff, const int *order, void *pre,
                      void *suf, int Jd, int *n_left, int *left, int *status, cudaStream_t s);
void launch_breakdown(const DevInst &I, const DevPop &P, int B, const double *lam, double *rt, double *out,
                      cudaStream_t s);

void launch_plan(const DevInst &I, const DevPop &P, const LsParams &L, cudaStream_t s);
void launch_eval(const DevInst &I, const DevPop &P, const LsParams &L, int grid, bool win, cudaStream_t s,
                 const cudaStream_t *side, cudaEvent_t *ev, cudaEvent_t *kt = nullptr);
void launch_eval_g(const DevInst &I, const DevPop &P, const LsParams &L, int grid, bool win, cudaStream_t s);
void launch_select(const DevInst &I, const DevPop &P, const LsParams &L, bool win, cudaStream_t s);
void launch_eval_mat(const DevInst &I, const DevPop &P, int b, int op, const MatCands &c, const double *lam,
                     MatDeltas out, bool win, cudaStream_t s);
void launch_emit(const DevInst &I, const DevPop &P, int b, int op, long long items, unsigned long long *keys,
                 cudaStream_t s);
void launch_totals(const DevInst &I, const DevPop &P, int b, double *out, cudaStream_t s);
void launch_lf_prep(const MatCands &c, const MatDeltas &d, unsigned long long *ord, unsigned long long *key,
                    unsigned char *flag, int *nan, cudaStream_t s);
int eval_grid_size(bool win);
void launch_route_sim(const DevInst &I, int nr, const int *off, const int *seq, int want_min, double *raw,
                      double *out, cudaStream_t s);
void launch_unpack(const DevInst &I, const DevPop &P, int B, const int *rbase, const int *coff, const int *cust,
                   const int *dep, const int *arr, cudaStream_t s);
void launch_pack(const DevPop &P, int b0, int B, int best, int *rbase, int *coff, int *cust, int *dep, int *arr, int *hdr,
                 int cap_r, int cap_c, cudaStream_t s);

struct XcPop {  // the population's members, flattened
  const int *mroute;  // [M+1] first route of member m
  const int *coff;    // [R+1] first customer of route r
  const int *cust;
  const int *dep, *arr;
};

struct XcJob {  // per offspring
  const int *main, *donors;  // [B], [B][M-1]
  uint32_t *mt;              // [B][625] state words + index (updated: the stream after the draws)
  const double *sig;         // [B][2] sigma_min, sigma_max
};

struct XcOut {
  int *refs;    // [B][Jcap] offspring routes as member routes (global route ids), then kept flags
  int *nref;    // [B]
  int *orig;    // [B][Jcap] 1 = main origin
  int *keep;    // [B][Ccap] per offspring customer slot (route order, position order): 1 kept
  int *unr;     // [B][NC] unrouted customers, ascending
  int *nunr;    // [B]
  double *sigma;  // [B]
  int *status;    // [B]
  int Jcap, Ccap;
};

void launch_exchange(const DevInst &I, const XcPop &X, const XcJob &Jb, const XcOut &O, int B, int M, int *prv,
                     int *nxt, int *owner, unsigned *bits, int *cnt, long long *key, int cnt_cap, cudaStream_t s);

}  // namespace mdr
