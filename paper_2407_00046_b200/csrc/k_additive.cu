// k_additive.cu -- NEXT-1 ablation: the two-level additive preconditioner of App. A (PAPER.md:730-749,
// "comparison only, not adopted"; DESIGN.md R-AS1):
//   M^-1 = sum_b B_b^T (B_b A B_b^T)^-1 B_b
// over level 1 = every node's 3x3 diagonal block (the block-Jacobi inverse D^-1 the PCG update
// applies anyway) and level 2 = aggregates of kAsAggNodes consecutive nodes (27x27 principal
// submatrices, the last aggregate ragged).  The level-2 inverses are computed once per Newton step
// by Gauss-Jordan elimination in shared memory, one CTA per aggregate; applying M^-1 is one
// dense 27x27 product per aggregate ("two block-wise SpMVs"), fused with the (r, u) partial of
// the single-reduction PCG.
#include "common.cuh"
#include "kernels.h"
#include "reduce.cuh"

namespace bal {

namespace {

constexpr int kAsDim = 3 * kAsAggNodes;  // 27
constexpr int kAsBuildThreads = 256;

// one CTA per aggregate: gather the principal submatrix (static full BSR + contact BSR), in-place
// Gauss-Jordan inversion without pivoting (A_agg is SPD: fixed nodes contribute identity rows, App. C),
// store the inverse [kAsDim][kAsDim] (ragged aggregates padded with zeros)
__global__ void __launch_bounds__(kAsBuildThreads)
k_as_build(int N, const int* __restrict__ srp, const int* __restrict__ scol, const double* __restrict__ sval,
           const int* __restrict__ crp, const int* __restrict__ ccol, const double* __restrict__ cval,
           double* __restrict__ inv, int* __restrict__ bad) {
  __shared__ double a[kAsDim][kAsDim + 1];
  __shared__ double fcol[kAsDim];
  const int ag = blockIdx.x, a0 = ag * kAsAggNodes;
  const int na = min(kAsAggNodes, N - a0), n = 3 * na;
  for (int e = threadIdx.x; e < kAsDim * kAsDim; e += blockDim.x) a[e / kAsDim][e % kAsDim] = 0.0;
  __syncthreads();
  // one thread per row of the aggregate: its static blocks, then its contact blocks, in column order
  if (threadIdx.x < na) {
    const int li = threadIdx.x, i = a0 + li;
    for (int pass = 0; pass < 2; ++pass) {
      const int* rp = pass ? crp : srp;
      if (!rp) continue;
      const int* cl = pass ? ccol : scol;
      const double* vl = pass ? cval : sval;
      for (int q = rp[i]; q < rp[i + 1]; ++q) {
        const int lj = cl[q] - a0;
        if (lj < 0 || lj >= na) continue;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) a[3 * li + r][3 * lj + c] += vl[9 * (size_t)q + 3 * r + c];
      }
    }
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const double piv = a[k][k];
    if (threadIdx.x == 0 && !(piv > 0.0)) atomicExch(bad, 1);  // not SPD (cannot happen for a PSD assembly)
    const double p = 1.0 / piv;
    if (threadIdx.x < n) fcol[threadIdx.x] = a[threadIdx.x][k];
    __syncthreads();
    // pivot row: a[k][j] *= p, a[k][k] = p
    if (threadIdx.x < n) a[k][threadIdx.x] = (threadIdx.x == k) ? p : a[k][threadIdx.x] * p;
    __syncthreads();
    // other rows: a[i][j] -= f_i a[k][j] (j != k), a[i][k] = -f_i p
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      if (i == k) continue;
      const double f = fcol[i];
      a[i][j] = (j == k) ? -f * p : a[i][j] - f * a[k][j];
    }
    __syncthreads();
  }
  double* o = inv + (size_t)ag * kAsDim * kAsDim;
  for (int e = threadIdx.x; e < kAsDim * kAsDim; e += blockDim.x) {
    const int i = e / kAsDim, j = e % kAsDim;
    o[e] = (i < n && j < n) ? a[i][j] : 0.0;
  }
}

// u += A_agg^-1 r_agg for every aggregate (u already holds D^-1 r), one warp per aggregate (lane l
// = row l of the aggregate); upart[2 b] += (r, A_agg^-1 r) of this block's aggregates (the level-2
// part of the PCG's (r, u); the level-1 part was written by the update / init kernel before)
__global__ void __launch_bounds__(kVecThreads)
k_as_apply(int N, int n_agg, const double* __restrict__ inv, const double* __restrict__ r, double* __restrict__ u,
           double* __restrict__ upart, const PcgScal* sc) {
  if (sc && sc->done) return;
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  double g = 0.0;
  for (int ag = wg; ag < n_agg; ag += nw) {
    const int a0 = ag * kAsAggNodes, n = 3 * min(kAsAggNodes, N - a0);
    const double rl = lane < n ? r[3 * (size_t)a0 + lane] : 0.0;
    const double* m = inv + (size_t)ag * kAsDim * kAsDim;
    double acc = 0.0;
    for (int c = 0; c < n; ++c) {  // column c of the (symmetric) inverse: coalesced
      const double rc = __shfl_sync(0xffffffffu, rl, c);
      if (lane < n) acc = fma(m[c * kAsDim + lane], rc, acc);
    }
    if (lane < n) {
      u[3 * (size_t)a0 + lane] += acc;
      g += rl * acc;
    }
  }
  __shared__ double sh[kVecThreads / 32];
  const double bg = block_sum<kVecThreads>(g, sh);
  if (threadIdx.x == 0) upart[2 * blockIdx.x] += bg;
}

}  // namespace

int as_num_aggregates(int N) { return (N + kAsAggNodes - 1) / kAsAggNodes; }

void launch_as_build(cudaStream_t st, int N, const int* srp, const int* scol, const double* sval, const int* crp,
                     const int* ccol, const double* cval, double* inv, int* bad) {
  const int na = as_num_aggregates(N);
  if (na == 0) return;
  k_as_build<<<na, kAsBuildThreads, 0, st>>>(N, srp, scol, sval, crp, ccol, cval, inv, bad);
  CK(cudaGetLastError());
}

void launch_as_apply(cudaStream_t st, int N, const double* inv, const double* r, double* u, double* upart,
                     const PcgScal* sc) {
  k_as_apply<<<kVecBlocks, kVecThreads, 0, st>>>(N, as_num_aggregates(N), inv, r, u, upart, sc);
  CK(cudaGetLastError());
}

}  // namespace bal
