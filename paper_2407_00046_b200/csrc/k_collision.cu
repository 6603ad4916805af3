// k_collision.cu -- constraint sets, barrier / AL energies and CCD.
//
//  * constraint_set: resolve every candidate feature pair at x (Q27), keep d < dhat,
//    canonical 128-bit keys, radix sort + unique (Q28), distance recomputed from the key.
//  * CCD: coplanarity cubic on [-eps, 1+eps], Newton-bisection on the monotone pieces
//    split at the roots of c'(t), deflation (Q31), activation d_TOC < eps + min(dhat, 1e-2 d_0) (R-CCD2; P:468's eps + dhat with BAL_CCD_LITERAL), conservative
//    TOI with the reference-frame sign test and x0.9 backtracking (fig:ccd_toi; DESIGN R-CCD1).
//  * energies: sigma * sum b(d; dhat) over C(x) and the A' terms mu (dhat + s - d) + sigma b(d; dhat + s)
//    (eq:aug-lag); deterministic fixed-order reductions.
#include <cub/cub.cuh>
#include <vector>

#include "bvh.h"
#include "geometry.cuh"
#include "kernels.h"

namespace bal {

constexpr double kCcdEps = 1e-12;  // P:468 "epsilon = 10^-12"

void broad_phase(cudaStream_t st, CollisionWork& w, Candidates& c, int V, const int* sverts, int F, const int* tris,
                 int E, const int* edges, const double* xa, const double* xb, double inflate, const uint8_t* fixed) {
  const double h = 0.5 * inflate;
  w.tri_tree.build(st, F, 3, tris, xa, xb, h);
  w.edge_tree.build(st, E, 2, edges, xa, xb, h);
  c.npt = query_pairs(st, w.tri_tree, 0, V, sverts, tris, xa, xb, h, fixed, c.pt, c.cnt);
  c.nee = query_pairs(st, w.edge_tree, 1, E, edges, edges, xa, xb, h, fixed, c.ee, c.cnt);
}

// ------------------------------------------------------------------ constraint set at x
__global__ void k_resolve_candidates(int n, int ftype, const int4* __restrict__ pairs, const double* __restrict__ x,
                                     double dhat2, unsigned long long* hi, unsigned long long* lo, int* idx,
                                     int* count, int cap) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int4 p = pairs[i];
  const Resolved r = resolve(ftype, ld3(x, p.x), ld3(x, p.y), ld3(x, p.z), ld3(x, p.w));
  if (!(r.D < dhat2)) return;
  // DESIGN.md R-DUP1: the constraint is the feature pair itself (key = PT|EE + role-ordered ids)
  Key k;
  k.t = ftype;
  k.n[0] = p.x;
  k.n[1] = p.y;
  k.n[2] = p.z;
  k.n[3] = p.w;
  const int s = atomicAdd(count, 1);
  if (s < cap) {
    hi[s] = key_hi(k);
    lo[s] = key_lo(k);
    idx[s] = s;
  }
}

// distance of a key's feature pair (re-resolving its sub-type at x)
BAL_D double key_dist(const Key& k, const double* __restrict__ x) {
  const int kn = type_nodes(k.t);
  d3 P[4];
  for (int a = 0; a < 4; ++a) P[a] = a < kn ? ld3(x, k.n[a]) : mk(0, 0, 0);
  return sqrt(resolve(k.t, P[0], P[1], P[2], P[3]).D);
}

__global__ void k_emit_unique(int nu, const int* __restrict__ start, const unsigned long long* __restrict__ hi,
                              const unsigned long long* __restrict__ lo, const double* __restrict__ x, int* keys5,
                              double* d, unsigned long long* uhi, unsigned long long* ulo) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nu) return;
  const int b = start[u];
  const Key k = key_from(hi[b], lo[b]);
  keys5[5 * (size_t)u] = k.t;
  for (int a = 0; a < 4; ++a) keys5[5 * (size_t)u + 1 + a] = k.n[a];
  d[u] = key_dist(k, x);
  uhi[u] = hi[b];
  ulo[u] = lo[b];
}

int constraint_set(cudaStream_t st, ConstraintSet& cs, const Candidates& c, const double* x, double dhat) {
  const int ncand = c.npt + c.nee;
  cs.n = 0;
  if (ncand == 0) return 0;
  KeySorter& ks = cs.ks;
  ks.prepare(ncand);
  cs.cnt.reserve(1);
  CK(cudaMemsetAsync(cs.cnt.ptr, 0, sizeof(int), st));
  const double d2 = dhat * dhat;
  if (c.npt)
    k_resolve_candidates<<<ceil_div(c.npt, 256), 256, 0, st>>>(c.npt, T_PT, c.pt.ptr, x, d2, ks.hi.ptr, ks.lo.ptr,
                                                                ks.idx.ptr, cs.cnt.ptr, ncand);
  if (c.nee)
    k_resolve_candidates<<<ceil_div(c.nee, 256), 256, 0, st>>>(c.nee, T_EE, c.ee.ptr, x, d2, ks.hi.ptr, ks.lo.ptr,
                                                                ks.idx.ptr, cs.cnt.ptr, ncand);
  CK(cudaGetLastError());
  int m = 0;
  CK(cudaMemcpyAsync(&m, cs.cnt.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (m == 0) return 0;
  ks.sort_packed(st, m);
  const int nu = ks.unique(st, m);
  cs.keys.reserve(5 * (size_t)nu);
  cs.d.reserve(nu);
  cs.hi.reserve(nu);
  cs.lo.reserve(nu);
  k_emit_unique<<<ceil_div(nu, 256), 256, 0, st>>>(nu, ks.start.ptr, ks.hi.ptr, ks.lo.ptr, x, cs.keys.ptr, cs.d.ptr,
                                                   cs.hi.ptr, cs.lo.ptr);
  CK(cudaGetLastError());
  cs.n = nu;
  return nu;
}

// ------------------------------------------------------------------ energies
__global__ void k_barrier_vals(int n, const double* __restrict__ d, double sigma, double dhat, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double di = d[i];
  out[i] = (di > 0.0) ? sigma * barrier_b(di, dhat) : INFINITY;
}

void barrier_energy(cudaStream_t st, CollisionWork& w, const ConstraintSet& cs, double sigma, double dhat,
                    double* out_sum, double* out_min) {
  if (cs.n == 0) {
    const double z[2] = {0.0, INFINITY};
    CK(cudaMemcpyAsync(out_sum, &z[0], sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(out_min, &z[1], sizeof(double), cudaMemcpyHostToDevice, st));
    return;
  }
  w.vals.reserve(cs.n);
  w.part.reserve(kRedBlocks);
  k_barrier_vals<<<ceil_div(cs.n, 256), 256, 0, st>>>(cs.n, cs.d.ptr, sigma, dhat, w.vals.ptr);
  launch_sum(st, cs.n, w.vals.ptr, w.part.ptr, out_sum);
  launch_min(st, cs.n, cs.d.ptr, w.part.ptr, out_min);
}

__global__ void k_key_dist(int n, const int* __restrict__ keys, const double* __restrict__ x, double* d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Key k;
  k.t = keys[5 * (size_t)i];
  for (int a = 0; a < 4; ++a) k.n[a] = keys[5 * (size_t)i + 1 + a];
  d[i] = key_dist(k, x);
}
void key_distances(cudaStream_t st, int n, const int* keys, const double* x, double* d) {
  if (n <= 0) return;
  k_key_dist<<<ceil_div(n, 256), 256, 0, st>>>(n, keys, x, d);
  CK(cudaGetLastError());
}

__global__ void k_phi_al(int n, const double* __restrict__ d, const double* __restrict__ mu,
                         const double* __restrict__ s, double sigma, double dhat, double* out, double* out_abs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double di = d[i];
  const double v = (di > 0.0) ? mu[i] * (dhat + s[i] - di) + sigma * barrier_b(di, dhat + s[i]) : INFINITY;
  out[i] = v;
  out_abs[i] = fabs(v);
}
void phi_al_energy(cudaStream_t st, CollisionWork& w, int n, const double* d, const double* mu, const double* s,
                   double sigma, double dhat, double* out_sum, double* out_min, double* out_abs_sum) {
  w.vals.reserve(2 * (size_t)std::max(n, 1));
  w.part.reserve(kRedBlocks);
  k_phi_al<<<ceil_div(n, 256), 256, 0, st>>>(n, d, mu, s, sigma, dhat, w.vals.ptr, w.vals.ptr + n);
  launch_sum(st, n, w.vals.ptr, w.part.ptr, out_sum);
  launch_sum(st, n, w.vals.ptr + n, w.part.ptr, out_abs_sum);
  launch_min(st, n, d, w.part.ptr, out_min);
}

// ------------------------------------------------------------------ CCD
BAL_D double cpoly(double a, double b, double c, double d, double t) { return ((a * t + b) * t + c) * t + d; }

BAL_D int quad_roots(double A, double B, double C, double r[2]) {
  if (A == 0.0) {
    if (B == 0.0) return 0;
    r[0] = -C / B;
    return 1;
  }
  const double disc = B * B - 4.0 * A * C;
  if (disc < 0.0) return 0;
  const double sq = sqrt(disc);
  const double q = -0.5 * (B + (B >= 0 ? sq : -sq));
  r[0] = q / A;
  if (q != 0.0) {
    r[1] = C / q;
    return 2;
  }
  return 1;
}

BAL_D double newton_bisect(double a, double b, double c, double d, double lo, double hi) {
  double flo = cpoly(a, b, c, d, lo);
  double t = 0.5 * (lo + hi);
  for (int it = 0; it < 100; ++it) {
    const double ft = cpoly(a, b, c, d, t);
    if (ft == 0.0) return t;
    if ((ft < 0) == (flo < 0)) {
      lo = t;
      flo = ft;
    } else {
      hi = t;
    }
    const double dft = (3.0 * a * t + 2.0 * b) * t + c;
    double tn = (dft != 0.0) ? t - ft / dft : 0.5 * (lo + hi);
    if (!(lo < tn && tn < hi)) tn = 0.5 * (lo + hi);
    if (fabs(tn - t) <= 1e-15) return tn;
    t = tn;
  }
  return t;
}

// roots in [lo, hi] clamped to [0,1] ascending; returns count (<= 3)
BAL_D int cubic_roots(double a, double b, double c, double d, double out[3]) {
  const double lo = -kCcdEps, hi = 1.0 + kCcdEps;
  double r[3];
  int nr = 0;
  if (a == 0.0) {
    nr = quad_roots(b, c, d, r);
  } else {
    double cr[2];
    int nc = quad_roots(3.0 * a, 2.0 * b, c, cr);
    double crit[2];
    int ncrit = 0;
    for (int i = 0; i < nc; ++i)
      if (lo < cr[i] && cr[i] < hi) crit[ncrit++] = cr[i];
    if (ncrit == 2 && crit[1] < crit[0]) {
      const double t = crit[0];
      crit[0] = crit[1];
      crit[1] = t;
    }
    double knots[4];
    int nk = 0;
    knots[nk++] = lo;
    for (int i = 0; i < ncrit; ++i) knots[nk++] = crit[i];
    knots[nk++] = hi;
    for (int i = 0; i + 1 < nk; ++i) {
      const double l = knots[i], h = knots[i + 1];
      const double fl = cpoly(a, b, c, d, l), fh = cpoly(a, b, c, d, h);
      double r1;
      if (fl == 0.0) r1 = l;
      else if (fh == 0.0) r1 = h;
      else if ((fl < 0) != (fh < 0)) r1 = newton_bisect(a, b, c, d, l, h);
      else continue;
      const double B = b + a * r1;
      const double C = c + B * r1;
      r[0] = r1;
      double q[2];
      const int nq = quad_roots(a, B, C, q);
      nr = 1;
      for (int k = 0; k < nq; ++k) r[nr++] = q[k];
      break;
    }
  }
  int n = 0;
  for (int i = 0; i < nr; ++i)
    if (lo <= r[i] && r[i] <= hi) out[n++] = fmin(fmax(r[i], 0.0), 1.0);
  // insertion sort
  for (int i = 1; i < n; ++i)
    for (int j = i; j > 0 && out[j] < out[j - 1]; --j) {
      const double t = out[j];
      out[j] = out[j - 1];
      out[j - 1] = t;
    }
  return n;
}

BAL_D double det3(d3 a, d3 b, d3 c) { return dot(a, cross(b, c)); }

BAL_D double signed_dist(int ftype, const d3 P[4]) {
  if (ftype == T_PT) return dot(P[0] - P[1], cross(P[2] - P[1], P[3] - P[1]));
  return dot(P[0] - P[2], cross(P[1] - P[0], P[3] - P[2]));
}

BAL_D double pair_toi(int ftype, const d3 X0[4], const d3 DX[4], double dhat, double d0frac) {
  const d3 e0[3] = {X0[1] - X0[0], X0[2] - X0[0], X0[3] - X0[0]};
  const d3 f[3] = {DX[1] - DX[0], DX[2] - DX[0], DX[3] - DX[0]};
  const double dd = det3(e0[0], e0[1], e0[2]);
  const double cc = det3(f[0], e0[1], e0[2]) + det3(e0[0], f[1], e0[2]) + det3(e0[0], e0[1], f[2]);
  const double bb = det3(f[0], f[1], e0[2]) + det3(f[0], e0[1], f[2]) + det3(e0[0], f[1], f[2]);
  const double aa = det3(f[0], f[1], f[2]);
  if (aa == 0.0 && bb == 0.0 && cc == 0.0 && dd == 0.0) {
    const double d0 = sqrt(resolve(ftype, X0[0], X0[1], X0[2], X0[3]).D);
    const int na = ftype == T_PT ? 1 : 2;
    double ma = 0.0, mb = 0.0;
    for (int k = 0; k < 4; ++k) {
      const double nk = sqrt(dot(DX[k], DX[k]));
      if (k < na) ma = fmax(ma, nk);
      else mb = fmax(mb, nk);
    }
    if (ma + mb == 0.0) return 1.0;
    return fmin(1.0, 0.9 * d0 / (ma + mb));
  }
  double roots[3];
  const int nr = cubic_roots(aa, bb, cc, dd, roots);
  if (nr == 0) return 1.0;
  // DESIGN.md R-CCD2: activation margin eps + min(dhat, 1e-2 d_0) (P:468 writes eps + dhat: the
  // literal reading is d0frac = +inf, flag BAL_CCD_LITERAL)
  const double d0 = sqrt(resolve(ftype, X0[0], X0[1], X0[2], X0[3]).D);
  const double thr = kCcdEps + fmin(dhat, d0frac * d0);
  double t_prev = 0.0;
  for (int i = 0; i < nr; ++i) {
    const double t = roots[i];
    d3 P[4];
    for (int k = 0; k < 4; ++k) P[k] = X0[k] + t * DX[k];
    const Resolved rs = resolve(ftype, P[0], P[1], P[2], P[3]);
    if (sqrt(rs.D) < thr) {
      double toi = 0.9 * t;
      if (rs.type == T_PT || rs.type == T_EE) {
        const double tref = 0.5 * (t_prev + t);
        d3 R[4];
        for (int k = 0; k < 4; ++k) R[k] = X0[k] + tref * DX[k];
        const bool sref = signed_dist(ftype, R) > 0;
        int n = 0;
        while (true) {
          d3 Q[4];
          for (int k = 0; k < 4; ++k) Q[k] = X0[k] + toi * DX[k];
          if ((signed_dist(ftype, Q) > 0) == sref) break;
          toi *= 0.9;
          if (toi <= t_prev) {  // DESIGN.md R-CCD3: crossed back over an earlier, non-contact root
            toi = tref;
            break;
          }
          if (++n >= 200) {
            toi = 0.0;
            break;
          }
        }
      }
      return toi;
    }
    t_prev = t;
  }
  return 1.0;
}

__global__ void k_ccd(int n, int ftype, const int4* __restrict__ pairs, const double* __restrict__ x,
                      const double* __restrict__ dx, double dhat, double d0frac, double* out) {
  __shared__ double sh[kRedThreads / 32];
  double tmin = 1.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int4 p = pairs[i];
    const int id[4] = {p.x, p.y, p.z, p.w};
    d3 X0[4], DX[4];
    for (int k = 0; k < 4; ++k) {
      X0[k] = ld3(x, id[k]);
      DX[k] = ld3(dx, id[k]);
    }
    tmin = fmin(tmin, pair_toi(ftype, X0, DX, dhat, d0frac));
  }
  tmin = block_min<kRedThreads>(tmin, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = tmin;
}

double ccd_step_toi(cudaStream_t st, CollisionWork& w, const Candidates& c, const double* x, const double* dx,
                    double dhat, double d0frac) {
  w.toi.reserve(2 * kRedBlocks + 2);
  w.part.reserve(kRedBlocks);
  const int nb = kRedBlocks;
  double* o = w.toi.ptr;
  // initialise both halves to 1.0 via a tiny fill of partials
  std::vector<double> ones(2 * nb, 1.0);
  CK(cudaMemcpyAsync(o, ones.data(), 2 * nb * sizeof(double), cudaMemcpyHostToDevice, st));
  if (c.npt) k_ccd<<<nb, kRedThreads, 0, st>>>(c.npt, T_PT, c.pt.ptr, x, dx, dhat, d0frac, o);
  if (c.nee) k_ccd<<<nb, kRedThreads, 0, st>>>(c.nee, T_EE, c.ee.ptr, x, dx, dhat, d0frac, o + nb);
  CK(cudaGetLastError());
  launch_min(st, 2 * nb, o, w.part.ptr, o + 2 * nb);
  double t = 1.0;
  CK(cudaMemcpyAsync(&t, o + 2 * nb, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return std::fmin(1.0, t);
}

}  // namespace bal
