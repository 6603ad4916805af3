// k_stencils.cu -- per-stencil gradients and PSD-projected Hessians.
//
//  K1 k_elastic : Neo-Hookean tet (Q1), closed-form P(F) and dP/dF, PSD projection of the
//                 12x12 DOF-space Hessian (Q21) done exactly on the 9-dim
//                 translation complement: H = (Q4 (x) I3) M (Q4 (x) I3)^T with the fixed
//                 Helmert basis Q4, M = V R^T (dP/dF) R (9x9), P(H) = (Q4 (x) I3) P(M) (...)^T.
//  K2 k_contact : barrier / augmented-Lagrangian stencil phi(d) (eq:aug-lag; Q22)
//                 with d = sqrt(D) and the envelope form of D = min_theta |r(x,theta)|^2:
//                 grad D = 2 w (x) r,  hess D = 2 (w w^T (x) I) - F_theta G^{-1} F_theta^T.
//  K3 k_friction: D_j = chi lam f(|P_n Gamma (x - x_t)|) (Q24-Q26), PSD by
//                 construction (no projection, not part of Lambda: Q17).
// Output per stencil: lower 3x3 blocks (a>=b, index a(a+1)/2+b) [n][10][9], gradient [n][12],
// lambda_bar = tr P(H) / (3k) [n]  (Q18).
// One thread per stencil; eigenvectors in shared memory [81][blockDim] (see psd.cuh).
#include "geometry.cuh"
#include "kernels.h"
#include "psd.cuh"

namespace bal {

// Helmert basis: Q[a][m], m < k-1: a <= m -> 1/sqrt((m+1)(m+2)); a == m+1 -> -(m+1)/sqrt(..)
BAL_HD double helmert(int a, int m) {
  const double s = 1.0 / sqrt((double)((m + 1) * (m + 2)));
  return a <= m ? s : (a == m + 1 ? -(double)(m + 1) * s : 0.0);
}

// expand packed P(M) (dim 3(k-1), index 3m+i) to the lower blocks of P(H) and write them
template <int K>
BAL_D void expand_write(const double (&PM)[Sym<3 * (K - 1)>::kSize], double* out /*[90]*/) {
  constexpr int NR = 3 * (K - 1);
  double Q[K][K - 1];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int m = 0; m < K - 1; ++m) Q[a][m] = helmert(a, m);
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b <= a; ++b) {
      double blk[9];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double s = 0.0;
#pragma unroll
          for (int m = 0; m < K - 1; ++m)
#pragma unroll
            for (int n = 0; n < K - 1; ++n) s += Q[a][m] * Q[b][n] * PM[Sym<NR>::id(3 * m + i, 3 * n + j)];
          blk[3 * i + j] = s;
        }
      double* o = out + 9 * (a * (a + 1) / 2 + b);
#pragma unroll
      for (int t = 0; t < 9; ++t) o[t] = blk[t];
    }
  for (int ab = K * (K + 1) / 2; ab < 10; ++ab)
    for (int t = 0; t < 9; ++t) out[9 * ab + t] = 0.0;
}

// Eigen-decomposition of a symmetric 3x3 matrix a (full, in/out: diagonalised) by cyclic Jacobi in
// registers; v: eigenvectors (columns).  Used for C = F^T F of ARAP tets (sigma_k^2 and V of the SVD).
BAL_D void sym3_eig(double (&a)[3][3], double (&v)[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) v[i][j] = (i == j) ? 1.0 : 0.0;
  const double fro2 = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2] +
                      2.0 * (a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2]);
  for (int sweep = 0; sweep < 20; ++sweep) {
    const double off2 = 2.0 * (a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2]);
    if (!(off2 > 1e-32 * fro2)) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      const double apq = a[p][q];
      if (apq == 0.0) continue;
      const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
      double t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
      if (theta < 0.0) t = -t;
      const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
#pragma unroll
      for (int k = 0; k < 3; ++k) {  // A <- A J (columns p, q)
        const double akp = a[k][p], akq = a[k][q];
        a[k][p] = c * akp - sn * akq;
        a[k][q] = sn * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {  // A <- J^T A (rows p, q)
        const double apk = a[p][k], aqk = a[q][k];
        a[p][k] = c * apk - sn * aqk;
        a[q][k] = sn * apk + c * aqk;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double vkp = v[k][p], vkq = v[k][q];
        v[k][p] = c * vkp - sn * vkq;
        v[k][q] = sn * vkp + c * vkq;
      }
    }
  }
}

// ARAP (NEXT-4, DESIGN.md R-ARAP): Psi = mu ||F - R||^2.  With C = F^T F = V diag(s^2) V^T (det V = 1)
// and U = F V diag(1/s): R = U V^T, dPsi/dF = 2 mu (F - R), and the F-space Hessian
// 2 mu (I - sum_{a<b} t_ab t_ab^T / (s_a + s_b)), t_ab = vec(u_a v_b^T - u_b v_a^T) (the twist modes).
struct ArapSvd {
  double s[3], U[3][3], V[3][3];
};
BAL_D ArapSvd arap_svd(const double (&F)[3][3]) {
  ArapSvd o;
  double Cm[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Cm[i][j] = F[0][i] * F[0][j] + F[1][i] * F[1][j] + F[2][i] * F[2][j];
  sym3_eig(Cm, o.V);
  const double dv = o.V[0][0] * (o.V[1][1] * o.V[2][2] - o.V[1][2] * o.V[2][1]) -
                    o.V[0][1] * (o.V[1][0] * o.V[2][2] - o.V[1][2] * o.V[2][0]) +
                    o.V[0][2] * (o.V[1][0] * o.V[2][1] - o.V[1][1] * o.V[2][0]);
  if (dv < 0.0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) o.V[k][2] = -o.V[k][2];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o.s[k] = sqrt(fmax(Cm[k][k], 0.0));
#pragma unroll
    for (int r = 0; r < 3; ++r)
      o.U[r][k] = (F[r][0] * o.V[0][k] + F[r][1] * o.V[1][k] + F[r][2] * o.V[2][k]) / o.s[k];
  }
  return o;
}

// ------------------------------------------------------------------------------------- K1
__global__ void __launch_bounds__(kElasticThreads)
k_elastic(int T, const double* __restrict__ x, const int4* __restrict__ tets,
          const double* __restrict__ Dm_inv, const double* __restrict__ vol,
          const double* __restrict__ mu_t, const double* __restrict__ lam_t, const unsigned char* __restrict__ model,
          double* __restrict__ stage, double* __restrict__ grad, double* __restrict__ lbar) {
  extern __shared__ double smem[];
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= T) return;
  double* V = smem + threadIdx.x;
  const int stride = blockDim.x;

  const int4 tt = tets[e];
  const d3 x0 = ld3(x, tt.x), x1 = ld3(x, tt.y), x2 = ld3(x, tt.z), x3 = ld3(x, tt.w);
  double Dm[3][3];
#pragma unroll
  for (int i = 0; i < 9; ++i) Dm[i / 3][i % 3] = Dm_inv[9 * (size_t)e + i];
  const double Ve = vol[e], mu = mu_t[e], lam = lam_t[e];
  const d3 c0 = x1 - x0, c1 = x2 - x0, c2v = x3 - x0;
  double Ds[3][3] = {{c0.x, c1.x, c2v.x}, {c0.y, c1.y, c2v.y}, {c0.z, c1.z, c2v.z}};
  double F[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) F[r][c] = Ds[r][0] * Dm[0][c] + Ds[r][1] * Dm[1][c] + Ds[r][2] * Dm[2][c];
  double C[3][3];  // cofactor matrix
  C[0][0] = F[1][1] * F[2][2] - F[1][2] * F[2][1];
  C[0][1] = F[1][2] * F[2][0] - F[1][0] * F[2][2];
  C[0][2] = F[1][0] * F[2][1] - F[1][1] * F[2][0];
  C[1][0] = F[0][2] * F[2][1] - F[0][1] * F[2][2];
  C[1][1] = F[0][0] * F[2][2] - F[0][2] * F[2][0];
  C[1][2] = F[0][1] * F[2][0] - F[0][0] * F[2][1];
  C[2][0] = F[0][1] * F[1][2] - F[0][2] * F[1][1];
  C[2][1] = F[0][2] * F[1][0] - F[0][0] * F[1][2];
  C[2][2] = F[0][0] * F[1][1] - F[0][1] * F[1][0];
  const double J = F[0][0] * C[0][0] + F[0][1] * C[0][1] + F[0][2] * C[0][2];
  const double lnJ = log(J);  // J <= 0 gives NaN: the line search never accepts such x
  double A[3][3];  // F^{-T}
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) A[i][j] = C[i][j] / J;
  const bool arap = model != nullptr && model[e] == 1;
  ArapSvd sv;
  double P[3][3];
  if (arap) {
    sv = arap_svd(F);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        P[i][j] = 2.0 * mu * (F[i][j] - (sv.U[i][0] * sv.V[j][0] + sv.U[i][1] * sv.V[j][1] + sv.U[i][2] * sv.V[j][2]));
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) P[i][j] = mu * (F[i][j] - A[i][j]) + lam * lnJ * A[i][j];
  }
  // gradient: dE/dDs = V P Dm^{-T}
  double G[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) G[r][c] = Ve * (P[r][0] * Dm[c][0] + P[r][1] * Dm[c][1] + P[r][2] * Dm[c][2]);
  double* g = grad + 12 * (size_t)e;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    g[r] = -(G[r][0] + G[r][1] + G[r][2]);
    g[3 + r] = G[r][0];
    g[6 + r] = G[r][1];
    g[9 + r] = G[r][2];
  }
  // shape-function gradients g_a (rows) and R3 = Q4^T Gamma
  double Gm[4][3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    Gm[1][j] = Dm[0][j];
    Gm[2][j] = Dm[1][j];
    Gm[3][j] = Dm[2][j];
    Gm[0][j] = -(Dm[0][j] + Dm[1][j] + Dm[2][j]);
  }
  double R3[3][3];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a) s += helmert(a, m) * Gm[a][j];
      R3[m][j] = s;
    }
  double S[3][3], B[3][3];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int n = 0; n < 3; ++n) S[m][n] = R3[m][0] * R3[n][0] + R3[m][1] * R3[n][1] + R3[m][2] * R3[n][2];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int n = 0; n < 3; ++n) B[i][n] = A[i][0] * R3[n][0] + A[i][1] * R3[n][1] + A[i][2] * R3[n][2];
  double M[Sym<9>::kSize];
  if (arap) {
    // reduced twist vectors w^{ab}_{(m,i)} = sum_j T_ab[i][j] R3[m][j], T_ab = u_a v_b^T - u_b v_a^T
    double W[3][9], cw[3];
#pragma unroll
    for (int ab = 0; ab < 3; ++ab) {
      const int a = ab == 2 ? 1 : 0, b = ab == 0 ? 1 : 2;
      cw[ab] = 1.0 / (sv.s[a] + sv.s[b]);
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < 3; ++j) t += (sv.U[i][a] * sv.V[j][b] - sv.U[i][b] * sv.V[j][a]) * R3[m][j];
          W[ab][3 * m + i] = t;
        }
    }
#pragma unroll
    for (int al = 0; al < 9; ++al)
#pragma unroll
      for (int be = al; be < 9; ++be) {
        const int m = al / 3, i = al % 3, n = be / 3, k = be % 3;
        const double tw = cw[0] * W[0][al] * W[0][be] + cw[1] * W[1][al] * W[1][be] + cw[2] * W[2][al] * W[2][be];
        M[Sym<9>::id(al, be)] = Ve * 2.0 * mu * ((i == k ? S[m][n] : 0.0) - tw);
      }
  } else {
    const double c2 = mu - lam * lnJ;
#pragma unroll
    for (int al = 0; al < 9; ++al)
#pragma unroll
      for (int be = al; be < 9; ++be) {
        const int m = al / 3, i = al % 3, n = be / 3, k = be % 3;
        M[Sym<9>::id(al, be)] =
            Ve * ((i == k ? mu * S[m][n] : 0.0) + c2 * B[i][n] * B[k][m] + lam * B[i][m] * B[k][n]);
      }
  }
  const double tr = psd_project<9>(M, V, stride);
  lbar[e] = tr / 12.0;
  expand_write<4>(M, stage + 90 * (size_t)e);
}

// Elastic energy per tet V Psi (Q1); +inf when J <= 0.
__global__ void k_elastic_energy(int T, const double* __restrict__ x, const int4* __restrict__ tets,
                                 const double* __restrict__ Dm_inv, const double* __restrict__ vol,
                                 const double* __restrict__ mu_t, const double* __restrict__ lam_t,
                                 const unsigned char* __restrict__ model, double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= T) return;
  const int4 tt = tets[e];
  const d3 x0 = ld3(x, tt.x), x1 = ld3(x, tt.y), x2 = ld3(x, tt.z), x3 = ld3(x, tt.w);
  double Dm[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) Dm[i] = Dm_inv[9 * (size_t)e + i];
  const d3 c0 = x1 - x0, c1 = x2 - x0, c2v = x3 - x0;
  double Ds[3][3] = {{c0.x, c1.x, c2v.x}, {c0.y, c1.y, c2v.y}, {c0.z, c1.z, c2v.z}};
  double F[3][3];
  double Ic = 0.0;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      F[r][c] = Ds[r][0] * Dm[c] + Ds[r][1] * Dm[3 + c] + Ds[r][2] * Dm[6 + c];
      Ic += F[r][c] * F[r][c];
    }
  const double J = F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) -
                   F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
                   F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
  if (!(J > 0.0)) {
    out[e] = INFINITY;
    return;
  }
  if (model != nullptr && model[e] == 1) {  // ARAP: mu (tr F^T F - 2 (s1 + s2 + s3) + 3)
    const ArapSvd sv = arap_svd(F);
    out[e] = vol[e] * mu_t[e] * (Ic - 2.0 * (sv.s[0] + sv.s[1] + sv.s[2]) + 3.0);
    return;
  }
  const double lnJ = log(J), mu = mu_t[e], lam = lam_t[e];
  out[e] = vol[e] * (0.5 * mu * (Ic - 3.0) - mu * lnJ + 0.5 * lam * lnJ * lnJ);
}

// ------------------------------------------------------------------------------------- K2
// Contact potential phi(d) and derivatives for one stencil (Q22).
BAL_D void phi_derivs(double d, double inA, double inAp, double mu, double s, double sigma, double dhat,
                      double& p1, double& p2) {
  p1 = 0.0;
  p2 = 0.0;
  if (inA != 0.0) {
    p1 += sigma * barrier_b1(d, dhat);
    p2 += sigma * barrier_b2(d, dhat);
  }
  if (inAp != 0.0) {
    p1 += -mu + sigma * barrier_b1(d, dhat + s);
    p2 += sigma * barrier_b2(d, dhat + s);
  }
}
BAL_HD double phi_value(double d, double inA, double inAp, double mu, double s, double sigma, double dhat) {
  double e = 0.0;
  if (inA != 0.0) e += sigma * barrier_b(d, dhat);
  if (inAp != 0.0) e += mu * (dhat + s - d) + sigma * barrier_b(d, dhat + s);
  return e;
}

// Envelope data of D = min_theta |r|^2 for a resolved sub-type: weights w (per key-local node),
// parameter directions E_p and their node coefficients c_p (per key-local node).
struct Envelope {
  d3 r;
  double w[4];
  int np;
  d3 E[2];
  double c[2][4];
};

BAL_D Envelope envelope(const Resolved& rs, const d3 P[4]) {
  Envelope ev;
  for (int a = 0; a < 4; ++a) {
    ev.w[a] = 0.0;
    ev.c[0][a] = 0.0;
    ev.c[1][a] = 0.0;
  }
  const int* L = rs.loc;
  if (rs.type == T_PP) {
    ev.r = P[L[0]] - P[L[1]];
    ev.w[L[0]] = 1.0;
    ev.w[L[1]] = -1.0;
    ev.np = 0;
  } else if (rs.type == T_PE) {
    const d3 p = P[L[0]], a = P[L[1]], b = P[L[2]];
    const d3 e = b - a;
    const double t = dot(p - a, e) / dot(e, e);
    ev.r = p - a - t * e;
    ev.w[L[0]] = 1.0;
    ev.w[L[1]] = -(1.0 - t);
    ev.w[L[2]] = -t;
    ev.np = 1;
    ev.E[0] = a - b;  // dr/dt = -e
    ev.c[0][L[1]] = 1.0;
    ev.c[0][L[2]] = -1.0;
  } else if (rs.type == T_PT) {
    const d3 p = P[L[0]], a = P[L[1]], b = P[L[2]], c = P[L[3]];
    const d3 e1 = b - a, e2 = c - a, w = p - a;
    const double a11 = dot(e1, e1), a12 = dot(e1, e2), a22 = dot(e2, e2);
    const double r1 = dot(e1, w), r2 = dot(e2, w);
    const double det = a11 * a22 - a12 * a12;
    const double u = (a22 * r1 - a12 * r2) / det;
    const double v = (a11 * r2 - a12 * r1) / det;
    ev.r = w - u * e1 - v * e2;
    ev.w[L[0]] = 1.0;
    ev.w[L[1]] = -(1.0 - u - v);
    ev.w[L[2]] = -u;
    ev.w[L[3]] = -v;
    ev.np = 2;
    ev.E[0] = a - b;  // dr/du = -e1
    ev.c[0][L[1]] = 1.0;
    ev.c[0][L[2]] = -1.0;
    ev.E[1] = a - c;  // dr/dv = -e2
    ev.c[1][L[1]] = 1.0;
    ev.c[1][L[3]] = -1.0;
  } else {
    const d3 a0 = P[L[0]], a1 = P[L[1]], b0 = P[L[2]], b1 = P[L[3]];
    const d3 ea = a1 - a0, eb = b1 - b0, rr = a0 - b0;
    const double a = dot(ea, ea), b = dot(ea, eb), c = dot(eb, eb);
    const double d = dot(ea, rr), e = dot(eb, rr);
    const double den = a * c - b * b;
    const double s = (b * e - c * d) / den;
    const double t = (a * e - b * d) / den;
    ev.r = rr + s * ea - t * eb;
    ev.w[L[0]] = 1.0 - s;
    ev.w[L[1]] = s;
    ev.w[L[2]] = -(1.0 - t);
    ev.w[L[3]] = -t;
    ev.np = 2;
    ev.E[0] = ea;  // dr/ds
    ev.c[0][L[0]] = -1.0;
    ev.c[0][L[1]] = 1.0;
    ev.E[1] = -1.0 * eb;  // dr/dt
    ev.c[1][L[2]] = 1.0;
    ev.c[1][L[3]] = -1.0;
  }
  return ev;
}

template <int K>
BAL_D double contact_hessian_project(const Envelope& ev, double alpha, double beta, double* V, int stride,
                                     double* out_blocks) {
  constexpr int NR = 3 * (K - 1);
  double wh[K - 1], ch[2][K - 1];
#pragma unroll
  for (int m = 0; m < K - 1; ++m) {
    double sw = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const double q = helmert(a, m);
      sw += q * ev.w[a];
      s0 += q * ev.c[0][a];
      s1 += q * ev.c[1][a];
    }
    wh[m] = sw;
    ch[0][m] = s0;
    ch[1][m] = s1;
  }
  const double r[3] = {ev.r.x, ev.r.y, ev.r.z};
  // G = 2 [E_p . E_q], Ginv
  double Gi[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  if (ev.np == 1) {
    Gi[0][0] = 1.0 / (2.0 * dot(ev.E[0], ev.E[0]));
  } else if (ev.np == 2) {
    const double g00 = 2.0 * dot(ev.E[0], ev.E[0]), g01 = 2.0 * dot(ev.E[0], ev.E[1]),
                 g11 = 2.0 * dot(ev.E[1], ev.E[1]);
    const double det = g00 * g11 - g01 * g01;
    Gi[0][0] = g11 / det;
    Gi[1][1] = g00 / det;
    Gi[0][1] = Gi[1][0] = -g01 / det;
  }
  double Fh[2][NR];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int m = 0; m < K - 1; ++m)
#pragma unroll
      for (int i = 0; i < 3; ++i)
        Fh[p][3 * m + i] = (p < ev.np) ? 2.0 * (wh[m] * comp(ev.E[p], i) + ch[p][m] * r[i]) : 0.0;
  double M[Sym<NR>::kSize];
#pragma unroll
  for (int al = 0; al < NR; ++al)
#pragma unroll
    for (int be = al; be < NR; ++be) {
      const int m = al / 3, i = al % 3, n = be / 3, j = be % 3;
      double schur = 0.0;
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int q = 0; q < 2; ++q) schur += Fh[p][al] * Gi[p][q] * Fh[q][be];
      M[Sym<NR>::id(al, be)] = 4.0 * alpha * wh[m] * r[i] * wh[n] * r[j] +
                               beta * ((i == j ? 2.0 * wh[m] * wh[n] : 0.0) - schur);
    }
  const double tr = psd_project<NR>(M, V, stride);
  expand_write<K>(M, out_blocks);
  return tr;
}

__global__ void __launch_bounds__(kElasticThreads)
k_contact(int n, const double* __restrict__ x, const int* __restrict__ keys /*[n][5]*/,
          const double* __restrict__ inA, const double* __restrict__ inAp,
          const double* __restrict__ mu, const double* __restrict__ s, double sigma, double dhat,
          double* __restrict__ stage, double* __restrict__ grad, double* __restrict__ lbar,
          int* __restrict__ nodes /*[n][4]*/, double* __restrict__ dist_out, double* __restrict__ dphi_out) {
  extern __shared__ double smem[];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* V = smem + threadIdx.x;
  const int stride = blockDim.x;
  const int* kk = keys + 5 * (size_t)i;
  const int t = kk[0];
  const int kf = type_nodes(t);
  d3 Pf[4];
  int ndf[4];
  for (int a = 0; a < 4; ++a) {
    ndf[a] = (a < kf) ? kk[1 + a] : -1;
    Pf[a] = (a < kf) ? ld3(x, ndf[a]) : mk(0, 0, 0);
  }
  const Resolved rf = resolve(t, Pf[0], Pf[1], Pf[2], Pf[3]);
  // stencil = support of the resolved sub-type, in role order (DESIGN.md R-DUP1)
  const int k = type_nodes(rf.type);
  d3 P[4];
  Resolved rs;
  rs.type = rf.type;
  rs.D = rf.D;
  for (int a = 0; a < 4; ++a) {
    const int src = (a < k) ? rf.loc[a] : -1;
    P[a] = src >= 0 ? Pf[src] : mk(0, 0, 0);
    rs.loc[a] = (a < k) ? a : -1;
    nodes[4 * (size_t)i + a] = src >= 0 ? ndf[src] : -1;
  }
  const double D = rs.D, d = sqrt(D);
  double p1, p2;
  phi_derivs(d, inA[i], inAp[i], mu[i], s[i], sigma, dhat, p1, p2);
  if (dist_out) dist_out[i] = d;
  if (dphi_out) dphi_out[i] = p1;
  const Envelope ev = envelope(rs, P);
  // grad phi = phi'(d) grad d = phi'/d (w (x) r)
  double* g = grad + 12 * (size_t)i;
  for (int a = 0; a < 4; ++a) {
    const double f = p1 / d * ev.w[a];
    g[3 * a] = f * ev.r.x;
    g[3 * a + 1] = f * ev.r.y;
    g[3 * a + 2] = f * ev.r.z;
  }
  const double alpha = p2 / (4.0 * D) - p1 / (4.0 * D * d);
  const double beta = p1 / (2.0 * d);
  double* ob = stage + 90 * (size_t)i;
  double tr;
  if (k == 4)
    tr = contact_hessian_project<4>(ev, alpha, beta, V, stride, ob);
  else if (k == 3)
    tr = contact_hessian_project<3>(ev, alpha, beta, V, stride, ob);
  else
    tr = contact_hessian_project<2>(ev, alpha, beta, V, stride, ob);
  lbar[i] = tr / (3.0 * k);
}

// ------------------------------------------------------------------------------------- K3
__global__ void k_friction(int n, const double* __restrict__ x, const double* __restrict__ xt,
                           const int* __restrict__ keys, const double* __restrict__ gam /*[n][4]*/,
                           const double* __restrict__ nrm /*[n][3]*/, const double* __restrict__ lam,
                           double chi, double eps, double* __restrict__ stage, double* __restrict__ grad,
                           double* __restrict__ lbar, int* __restrict__ nodes) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int* kk = keys + 5 * (size_t)i;
  const int k = type_nodes(kk[0]);
  const d3 nn = mk(nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]);
  d3 u = mk(0, 0, 0);
  double G[4];
  for (int a = 0; a < 4; ++a) {
    G[a] = (a < k) ? gam[4 * (size_t)i + a] : 0.0;
    nodes[4 * (size_t)i + a] = (a < k) ? kk[1 + a] : -1;
    if (a < k) u = u + G[a] * (ld3(x, kk[1 + a]) - ld3(xt, kk[1 + a]));
  }
  const d3 w = u - dot(u, nn) * nn;
  const double y = sqrt(dot(w, w));
  double fpy, fpp;
  if (y < eps) {
    fpy = 2.0 / eps - y / (eps * eps);
    fpp = 2.0 / eps - 2.0 * y / (eps * eps);
  } else {
    fpy = 1.0 / y;
    fpp = 0.0;
  }
  const double cl = chi * lam[i];
  double* g = grad + 12 * (size_t)i;
  for (int a = 0; a < 4; ++a) {
    const double f = cl * fpy * G[a];
    g[3 * a] = f * w.x;
    g[3 * a + 1] = f * w.y;
    g[3 * a + 2] = f * w.z;
  }
  // K3 = fpy P_n + (fpp - fpy) what what^T
  const double nv[3] = {nn.x, nn.y, nn.z};
  const double wv[3] = {w.x, w.y, w.z};
  double K3[3][3];
  const double q = (y > 0.0) ? (fpp - fpy) / (y * y) : 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) K3[r][c] = fpy * ((r == c ? 1.0 : 0.0) - nv[r] * nv[c]) + q * wv[r] * wv[c];
  double* ob = stage + 90 * (size_t)i;
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b <= a; ++b) {
      const double f = cl * G[a] * G[b];
      for (int t = 0; t < 9; ++t) ob[9 * (a * (a + 1) / 2 + b) + t] = f * K3[t / 3][t % 3];
    }
  lbar[i] = 0.0;
}

__global__ void k_friction_energy(int n, const double* __restrict__ x, const double* __restrict__ xt,
                                  const int* __restrict__ keys, const double* __restrict__ gam,
                                  const double* __restrict__ nrm, const double* __restrict__ lam, double chi,
                                  double eps, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int* kk = keys + 5 * (size_t)i;
  const int k = type_nodes(kk[0]);
  const d3 nn = mk(nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]);
  d3 u = mk(0, 0, 0);
  for (int a = 0; a < k; ++a) u = u + gam[4 * (size_t)i + a] * (ld3(x, kk[1 + a]) - ld3(xt, kk[1 + a]));
  const d3 w = u - dot(u, nn) * nn;
  const double y = sqrt(dot(w, w));
  const double f = (y < eps) ? (-(y * y * y) / (3.0 * eps * eps) + y * y / eps) : (y - eps / 3.0);
  out[i] = chi * lam[i] * f;
}

// ------------------------------------------------------------------------------- launchers
size_t elastic_smem(int threads) { return sizeof(double) * 81 * (size_t)threads; }

void launch_elastic(cudaStream_t st, int T, const double* x, const int4* tets, const double* Dm_inv,
                    const double* vol, const double* mu, const double* lam, const unsigned char* model,
                    double* stage, double* grad, double* lbar) {
  if (T <= 0) return;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_elastic, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)elastic_smem(kElasticThreads)));
    CK(cudaFuncSetAttribute(k_contact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)elastic_smem(kElasticThreads)));
    attr = true;
  }
  k_elastic<<<ceil_div(T, kElasticThreads), kElasticThreads, elastic_smem(kElasticThreads), st>>>(
      T, x, tets, Dm_inv, vol, mu, lam, model, stage, grad, lbar);
  CK(cudaGetLastError());
}

void launch_elastic_energy(cudaStream_t st, int T, const double* x, const int4* tets, const double* Dm_inv,
                           const double* vol, const double* mu, const double* lam, const unsigned char* model,
                           double* out) {
  if (T <= 0) return;
  k_elastic_energy<<<ceil_div(T, 256), 256, 0, st>>>(T, x, tets, Dm_inv, vol, mu, lam, model, out);
  CK(cudaGetLastError());
}

void launch_contact(cudaStream_t st, int n, const double* x, const int* keys, const double* inA,
                    const double* inAp, const double* mu, const double* s, double sigma, double dhat,
                    double* stage, double* grad, double* lbar, int* nodes, double* dist, double* dphi) {
  if (n <= 0) return;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_contact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)elastic_smem(kElasticThreads)));
    attr = true;
  }
  k_contact<<<ceil_div(n, kElasticThreads), kElasticThreads, elastic_smem(kElasticThreads), st>>>(
      n, x, keys, inA, inAp, mu, s, sigma, dhat, stage, grad, lbar, nodes, dist, dphi);
  CK(cudaGetLastError());
}

void launch_friction(cudaStream_t st, int n, const double* x, const double* xt, const int* keys,
                     const double* gam, const double* nrm, const double* lam, double chi, double eps,
                     double* stage, double* grad, double* lbar, int* nodes) {
  if (n <= 0) return;
  k_friction<<<ceil_div(n, 128), 128, 0, st>>>(n, x, xt, keys, gam, nrm, lam, chi, eps, stage, grad, lbar,
                                               nodes);
  CK(cudaGetLastError());
}

void launch_friction_energy(cudaStream_t st, int n, const double* x, const double* xt, const int* keys,
                            const double* gam, const double* nrm, const double* lam, double chi, double eps,
                            double* out) {
  if (n <= 0) return;
  k_friction_energy<<<ceil_div(n, 128), 128, 0, st>>>(n, x, xt, keys, gam, nrm, lam, chi, eps, out);
  CK(cudaGetLastError());
}

}  // namespace bal
