// mdr_feasibility.cu -- the forward-simulation feasibility check on the device
// (reference model.py:242-392).
//
// One warp per route.  Lane 0 runs the earliest-departure simulation
// (simulate_from at t0 = e[first], model.py:242-282: wait for early windows,
// clamp late arrivals and carry the overshoot as time warp) and records the
// prefix of raw travel+service times; the lanes then split the departure-time
// candidates of minimal_duration (model.py:291-314: e/l of the first node and
// every window bound minus the raw time to reach it), simulate each one
// independently and keep the minimal duration among the warp-minimal
// candidates (a warp min; min is order-free).  Every expression keeps the
// reference's operation order (-fmad=false), so results are bit-identical.
#include "mdr_kernels.cuh"

namespace mdr {

struct Sim {
  double dist, load, dur, tw;
  int late;
};

__device__ Sim simulate_seq(const DevInst &I, const int *seq, int n, double t0) {
  Sim s{0.0, 0.0, 0.0, 0.0, 0};
  const int f = seq[0];
  const double4 nf = I.node[f];
  double start = nf.z > t0 ? nf.z : t0;  // Python max(t0, e): t0 unless e is larger
  if (start > nf.w) {
    s.tw += start - nf.w;
    s.late += 1;
    start = nf.w;
  }
  double now = start + nf.y;
  for (int i = 0; i + 1 < n; i++) {
    const int a = seq[i], b = seq[i + 1];
    const size_t k = (size_t)a * I.N + b;
    s.dist += I.dist[k];
    double arrive = now + (I.talias ? I.dist[k] : I.time[k]);
    const double4 nb = I.node[b];
    if (arrive < nb.z) {
      arrive = nb.z;
    } else if (arrive > nb.w) {
      s.tw += arrive - nb.w;
      s.late += 1;
      arrive = nb.w;
    }
    now = arrive + nb.y;
    s.load += nb.x;
  }
  s.dur = (now - start) + s.tw;
  return s;
}

// out[r*6 ..] = {distance, load, duration, time_warp, late_count, minimal duration}
__global__ void k_route_sim(DevInst I, int nr, const int *off, const int *seq, int want_min, double *raw,
                            double *out) {
  const int lane = threadIdx.x & 31;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nr) return;
  const int o = off[r], n = off[r + 1] - o;
  const int *sq = seq + o;
  double *rw = raw + o;
  Sim base{0.0, 0.0, 0.0, 0.0, 0};
  if (lane == 0) {
    base = simulate_seq(I, sq, n, I.node[sq[0]].z);
    double acc = 0.0;  // raw += s[a] + t[a, b] (model.py:300-301)
    for (int i = 0; i + 1 < n; i++) {
      const size_t k = (size_t)sq[i] * I.N + sq[i + 1];
      acc = acc + (I.node[sq[i]].y + (I.talias ? I.dist[k] : I.time[k]));
      rw[i] = acc;
    }
  }
  __syncwarp();
  base.dur = __shfl_sync(0xffffffffu, base.dur, 0);
  base.tw = __shfl_sync(0xffffffffu, base.tw, 0);
  double best = base.dur;
  if (want_min && I.win) {
    const double e0 = I.node[sq[0]].z;
    const int nc = 2 + 2 * (n - 1);
    for (int c = lane; c < nc; c += 32) {
      double t0;
      if (c < 2) {
        t0 = c == 0 ? e0 : I.node[sq[0]].w;
      } else {
        const int i = (c - 2) >> 1;
        const double4 nb = I.node[sq[i + 1]];
        t0 = ((c - 2) & 1 ? nb.w : nb.z) - rw[i];
        if (isinf((c - 2) & 1 ? nb.w : nb.z)) continue;
      }
      if (isinf(t0) || t0 < e0) continue;
      const Sim s = simulate_seq(I, sq, n, t0);
      if (s.tw <= base.tw + 1e-9 && s.dur < best) best = s.dur;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, best, s);
      if (x < best) best = x;
    }
  }
  if (lane == 0) {
    double *q = out + (size_t)r * 6;
    q[0] = base.dist;
    q[1] = base.load;
    q[2] = base.dur;
    q[3] = base.tw;
    q[4] = (double)base.late;
    q[5] = best;
  }
}

void launch_route_sim(const DevInst &I, int nr, const int *off, const int *seq, int want_min, double *raw,
                      double *out, cudaStream_t s) {
  if (nr <= 0) return;
  k_route_sim<<<(nr * 32 + 255) / 256, 256, 0, s>>>(I, nr, off, seq, want_min, raw, out);
}

}  // namespace mdr
