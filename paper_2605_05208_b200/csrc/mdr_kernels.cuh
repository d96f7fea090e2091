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

}  // namespace mdr
