// psd.cuh -- per-thread PSD projection of a small symmetric matrix (§4.2.2:
// "projecting the local Hessian to the closest symmetric positive semi-definite form" by
// "eliminating negative eigenvalues").
//
// B200 design: one thread owns one stencil.  The reduced matrix (translation null space
// removed exactly with a fixed Helmert basis, see k_stencils.cu) is at most 9x9; its upper
// triangle lives in registers (45 doubles, fully unrolled compile-time indices) and the
// eigenvector matrix in shared memory laid out [entry][thread] so a warp's accesses hit 32
// consecutive 8-byte words (conflict-free).  Cyclic Jacobi with the off-norm computed directly
// (never as ||A||^2 - ||diag||^2, which cancels) until off(A) <= 1e-15 ||A||_F or 30 sweeps.
#pragma once
#include "common.cuh"

namespace bal {

template <int N>
struct Sym {
  static constexpr int kSize = N * (N + 1) / 2;
  // upper-triangle packed index (i <= j)
  static BAL_HD constexpr int id(int i, int j) {
    return i <= j ? (i * N - i * (i - 1) / 2 + (j - i)) : (j * N - j * (j - 1) / 2 + (i - j));
  }
};

// A: packed symmetric matrix (in/out: on exit holds P(A), packed).  V: this thread's slice of a
// shared [N*N][stride] array.  Returns the sum of the clamped eigenvalues (= tr P(A)).
template <int N>
__device__ __forceinline__ double psd_project(double (&A)[Sym<N>::kSize], double* V, int stride) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) V[(i * N + j) * stride] = (i == j) ? 1.0 : 0.0;

  double fro2 = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i; j < N; ++j) {
      const double a = A[Sym<N>::id(i, j)];
      fro2 += (i == j ? 1.0 : 2.0) * a * a;
    }
  const double tol2 = 1e-30 * fro2;  // (1e-15 ||A||_F)^2

  for (int sweep = 0; sweep < 30; ++sweep) {
    double off2 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i + 1; j < N; ++j) off2 += 2.0 * A[Sym<N>::id(i, j)] * A[Sym<N>::id(i, j)];
    if (!(off2 > tol2)) break;
#pragma unroll
    for (int p = 0; p < N - 1; ++p) {
#pragma unroll
      for (int q = p + 1; q < N; ++q) {
        const double apq = A[Sym<N>::id(p, q)];
        if (apq != 0.0) {
          const double app = A[Sym<N>::id(p, p)], aqq = A[Sym<N>::id(q, q)];
          const double theta = (aqq - app) / (2.0 * apq);
          double t;
          if (fabs(theta) > 1e150) {
            t = 0.5 / theta;
          } else {
            t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
            if (theta < 0.0) t = -t;
          }
          const double c = 1.0 / sqrt(t * t + 1.0);
          const double s = t * c;
          A[Sym<N>::id(p, p)] = app - t * apq;
          A[Sym<N>::id(q, q)] = aqq + t * apq;
          A[Sym<N>::id(p, q)] = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            if (k != p && k != q) {
              const double akp = A[Sym<N>::id(k, p)], akq = A[Sym<N>::id(k, q)];
              A[Sym<N>::id(k, p)] = c * akp - s * akq;
              A[Sym<N>::id(k, q)] = s * akp + c * akq;
            }
          }
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const double vkp = V[(k * N + p) * stride], vkq = V[(k * N + q) * stride];
            V[(k * N + p) * stride] = c * vkp - s * vkq;
            V[(k * N + q) * stride] = s * vkp + c * vkq;
          }
        }
      }
    }
  }
  double lam[N];
  double tr = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    lam[k] = fmax(A[Sym<N>::id(k, k)], 0.0);
    tr += lam[k];
  }
  // P = V diag(lam+) V^T (upper triangle), exactly symmetric by construction
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i; j < N; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) s += V[(i * N + k) * stride] * lam[k] * V[(j * N + k) * stride];
      A[Sym<N>::id(i, j)] = s;
    }
  return tr;
}

}  // namespace bal
