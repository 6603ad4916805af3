// reduce.cuh -- deterministic reductions and PCG helpers shared by the single-GPU (k_linalg.cu) and
// the partitioned (pcg_dist.cu) block-Jacobi PCG: fixed grids, per-block partials, the last block
// reduces them in a fixed order (atomic ticket), per-group warp-match accumulation for the warm start.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace bal {

constexpr int kVecThreads = 256;
constexpr int kVecBlocks = 4 * kSMs;

BAL_D void dinv_apply(const double* __restrict__ dinv, int i, double r0, double r1, double r2, double& z0,
                      double& z1, double& z2) {
  const double* m = dinv + 6 * (size_t)i;
  z0 = m[0] * r0 + m[1] * r1 + m[2] * r2;
  z1 = m[1] * r0 + m[3] * r1 + m[4] * r2;
  z2 = m[2] * r0 + m[4] * r1 + m[5] * r2;
}

// last-block finalisation helper for NQ quantities
template <int NQ, int NT>
BAL_D bool last_block_reduce(const double (&loc)[NQ], double* partials, unsigned* counter, double (&tot)[NQ]) {
  __shared__ double sh[NT / 32];
  __shared__ bool last;
  double bs[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) bs[q] = block_sum<NT>(loc[q], sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) partials[NQ * blockIdx.x + q] = bs[q];
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double t = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t += partials[NQ * i + q];
    tot[q] = block_sum<NT>(t, sh);
  }
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

// App. B stop logic (oracle.linalg.pcg_run order): NaN, converged, stagnation, cap.
BAL_D void pcg_stop_check(PcgScal* sc, const double* hist) {
  const int k = sc->k;
  const double rn = hist[k];
  if (!isfinite(rn)) {
    sc->stop = 3;
    sc->done = 1;
    return;
  }
  const double thr = sc->crit == 2 ? sc->ukappa * sqrt(sc->xx) : sc->tol * sc->bnorm;
  if (rn <= thr) {
    sc->stop = 0;
    sc->done = 1;
    return;
  }
  // R-PCG1: stagnation = the CG objective (monotone in PCG) decreased by no more than kStallRel of
  // its total decrease over the last W iterations
  const int W = sc->window;
  if (W > 0 && k >= W) {
    bool stall;
    if (sc->lit) {  // literal P:757 / Q15: the best residual of the last W iterations is no better
      sc->pmin = fmin(sc->pmin, hist[k - W]);  // than the best before them
      double wmin = rn;
      for (int j = k - W + 1; j < k; ++j) wmin = fmin(wmin, hist[j]);
      stall = wmin >= sc->pmin;
    } else {  // R-PCG1
      const double* dh = hist + sc->hcap;
      stall = dh[k] - dh[k - W] <= sc->stall_rel * dh[k];
    }
    if (stall) {
      sc->stop = 1;
      sc->done = 1;
      return;
    }
  }
  if (k >= sc->max_iters) {
    sc->stop = 2;
    sc->done = 1;
  }
}

// Chronopoulos-Gear (single-reduction) PCG scalars, set by the last CTA of the SpMV kernel of
// iteration k (k_spmv_ts.cu) from gam = (r_k, u_k), rr = (r_k, r_k), delta = (A u_k, u_k), u = M^-1 r:
// App. B stop test on ||r_k|| (same order as pcg_stop_check for the textbook recurrences), then
// beta_k = gam_k / gam_{k-1}, alpha_k = gam_k / (delta_k - beta_k gam_k / alpha_{k-1}) -- computed
// even when the solve stops, so an App. B resume continues with the update of step k.  The CG
// objective decreases by alpha_{k-1} gam_{k-1} / 2 in step k-1 (R-PCG1 bookkeeping).
BAL_D void cg_scalars(PcgScal* sc, double* hist, double gam, double rr, double delta, double xx = 0.0) {
  const int k = sc->k;
  sc->xx = xx;
  if (k > 0) sc->dec += 0.5 * sc->alpha * sc->rz;
  sc->rr = rr;
  hist[k] = sqrt(rr);
  hist[sc->hcap + k] = sc->dec;
  pcg_stop_check(sc, hist);
  const double beta = (k > 0 && sc->rz != 0.0) ? gam / sc->rz : 0.0;
  const double den = (k > 0 && sc->alpha != 0.0) ? delta - beta * gam / sc->alpha : delta;
  sc->beta = beta;
  sc->pq = den;
  sc->alpha = (den != 0.0) ? gam / den : 0.0;  // r = 0 exactly: converged, the stop test fired
  sc->rz = gam;
}

template <int NQ>
BAL_D void grp_warp_accum(int g, const double (&v)[NQ], double* bucket /*[warps][kMaxGroups][NQ]*/) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned pending = __ballot_sync(0xffffffffu, g >= 0);
  while (pending) {
    const int leader = __ffs(pending) - 1;
    const int gl = __shfl_sync(0xffffffffu, g, leader);
    const unsigned members = __ballot_sync(0xffffffffu, g == gl);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double s = (g == gl) ? v[q] : 0.0;
      s = warp_sum(s);
      if (lane == leader) bucket[(w * kMaxGroups + gl) * NQ + q] += s;
    }
    pending &= ~members;
  }
}

// block buckets -> per-block partials [blk][kMaxGroups][NQ]; last block -> totals (thread g)
template <int NQ>
BAL_D bool grp_finish(double* bucket, double* partials, unsigned* counter, int G, double (&tot)[NQ]) {
  __shared__ bool last;
  constexpr int W = kVecThreads / 32;
  __syncthreads();
  for (int t = threadIdx.x; t < G * NQ; t += blockDim.x) {
    const int g = t / NQ, q = t % NQ;
    double s = 0.0;
    for (int w = 0; w < W; ++w) s += bucket[(w * kMaxGroups + g) * NQ + q];
    partials[((size_t)blockIdx.x * kMaxGroups + g) * NQ + q] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return false;
  __threadfence();
  if (threadIdx.x < G) {
    const int g = threadIdx.x;
    for (int q = 0; q < NQ; ++q) {
      double s = 0.0;
      for (int b = 0; b < (int)gridDim.x; ++b) s += partials[((size_t)b * kMaxGroups + g) * NQ + q];
      tot[q] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

BAL_D void ws_zero_bucket(double* bucket, int nq) {
  for (int t = threadIdx.x; t < (kVecThreads / 32) * kMaxGroups * nq; t += blockDim.x) bucket[t] = 0.0;
  __syncthreads();
}

}  // namespace bal
