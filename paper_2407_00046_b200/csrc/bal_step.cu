// bal_step.cu -- the barrier-augmented Lagrangian time step (Alg. 1) with its inexact
// Newton-PCG primal solve (§4); host orchestration of the device kernels, mirroring
// oracle/bal.py step by step.  Only per-Newton-iteration scalars cross
// to the host (||e||, alpha_CCD, line-search energies, counts).
#include <chrono>
#include <cmath>
#include <cstring>

#include <cub/cub.cuh>

#include "bvh.h"
#include "ctx.h"
#include "geometry.cuh"

using namespace bal;

struct StepWork {
  DevBuf<double> x, xn, dir, rhs, trial, gE, gb, v;
  Candidates cand_prox, cand_sw;
  ConstraintSet cs_A, cs_trial;
  CollisionWork cw;
  // A' (sorted by key): keys5, packed keys, multipliers, slacks, distances
  DevBuf<int> ap_keys, ap_keys_new;
  DevBuf<unsigned long long> ap_hi, ap_lo, ap_hi_new, ap_lo_new;
  DevBuf<double> ap_mu, ap_s, ap_mu_new, ap_s_new, ap_d;
  int n_ap = 0;
  DevBuf<double> evals, esc;  // per-item energies, energy scalars
  DevBuf<int> sel, selcnt;
  DevBuf<unsigned char> tmp;
  // state of the frame in progress (Alg. 1 loop variables), so the loop can be advanced in slices
  struct Frame {
    bool active = false, converged = false;
    int l = 0;
    double sigma = 0, sig0 = 0, dmin = 0, dmin_prev = 0, e0 = -1;
    // R-FRIC1: history of min ||e|| for the friction-anchor freeze
    std::vector<double> emin;
    bool fric_frozen = false;
    bal_step_stats S{};
    std::chrono::steady_clock::time_point t_start;
  } fr;
};

void destroy_step_work(bal_ctx* c) {
  delete c->sw;
  c->sw = nullptr;
}

namespace {

__global__ void k_predictor(int n, const double* __restrict__ xt, const double* __restrict__ vt, double h, double gx,
                            double gy, double gz, const uint8_t* __restrict__ fixed, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double g[3] = {gx, gy, gz};
  for (int c = 0; c < 3; ++c) {
    const size_t j = 3 * (size_t)i + c;
    y[j] = fixed[i] ? xt[j] : xt[j] + h * vt[j] + h * h * g[c];
  }
}

__global__ void k_inertia_energy(int n, const double* __restrict__ x, const double* __restrict__ y,
                                 const double* __restrict__ mass, double inv_2h2, const uint8_t* __restrict__ fixed,
                                 double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (fixed[i]) {
    out[i] = 0.0;
    return;
  }
  double s = 0.0;
  for (int c = 0; c < 3; ++c) {
    const double d = x[3 * (size_t)i + c] - y[3 * (size_t)i + c];
    s += d * d;
  }
  out[i] = mass[i] * s * inv_2h2;
}

__global__ void k_flag_lt(int n, const double* __restrict__ d, double thr, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = d[i] < thr ? 1 : 0;
}

__global__ void k_compact_keys(int n, const int* __restrict__ flag, const int* __restrict__ pos,
                               const int* __restrict__ keys, const unsigned long long* __restrict__ hi,
                               const unsigned long long* __restrict__ lo, int* okeys, unsigned long long* ohi,
                               unsigned long long* olo) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  const int p = pos[i];
  for (int a = 0; a < 5; ++a) okeys[5 * (size_t)p + a] = keys[5 * (size_t)i + a];
  ohi[p] = hi[i];
  olo[p] = lo[i];
}

// carry (mu, s) of surviving A' members by key; new members start at 0 (Q10)
__global__ void k_carry(int n, const unsigned long long* __restrict__ hi, const unsigned long long* __restrict__ lo,
                        int nold, const unsigned long long* __restrict__ ohi, const unsigned long long* __restrict__ olo,
                        const double* __restrict__ omu, const double* __restrict__ os, double* mu, double* s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int a = 0, b = nold;
  const unsigned long long h = hi[i], l = lo[i];
  while (a < b) {
    const int m = (a + b) >> 1;
    if (ohi[m] < h || (ohi[m] == h && olo[m] < l)) a = m + 1;
    else b = m;
  }
  const bool found = a < nold && ohi[a] == h && olo[a] == l;
  mu[i] = found ? omu[a] : 0.0;
  s[i] = found ? os[a] : 0.0;
}

// slack and multiplier update on A' (Alg. 1 lines 12-14)
__global__ void k_al_update(int n, const double* __restrict__ d, double sigma, double dhat, double* mu, double* s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double sn = fmax(-mu[i] / sigma - dhat + d[i], 0.0);
  s[i] = sn;
  mu[i] = mu[i] + sigma * barrier_b(d[i], dhat + sn);
}

// friction anchors per stencil of A u A' (Q25, Q26): Gamma, n at x; lambda = -phi'(d) for A members
__global__ void k_friction_anchor(int n, const int* __restrict__ keys, const double* __restrict__ inA,
                                  const double* __restrict__ inAp, const double* __restrict__ mu,
                                  const double* __restrict__ s, double sigma, double dhat,
                                  const double* __restrict__ x, double* gam, double* nrm, double* lam) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int t = keys[5 * (size_t)i];
  const int k = type_nodes(t);
  d3 P[4];
  for (int a = 0; a < 4; ++a) P[a] = a < k ? ld3(x, keys[5 * (size_t)i + 1 + a]) : mk(0, 0, 0);
  const Resolved rs = resolve(t, P[0], P[1], P[2], P[3]);
  double w[4] = {0, 0, 0, 0};
  const int* L = rs.loc;
  if (rs.type == T_PP) {
    w[L[0]] = 1.0;
    w[L[1]] = -1.0;
  } else if (rs.type == T_PE) {
    const d3 p = P[L[0]], a = P[L[1]], b = P[L[2]];
    const double tt = dot(p - a, b - a) / dot(b - a, b - a);
    w[L[0]] = 1.0;
    w[L[1]] = -(1.0 - tt);
    w[L[2]] = -tt;
  } else if (rs.type == T_PT) {
    const d3 p = P[L[0]], a = P[L[1]], b = P[L[2]], c = P[L[3]];
    const d3 e1 = b - a, e2 = c - a, ww = p - a;
    const double a11 = dot(e1, e1), a12 = dot(e1, e2), a22 = dot(e2, e2);
    const double det = a11 * a22 - a12 * a12;
    const double u = (a22 * dot(e1, ww) - a12 * dot(e2, ww)) / det;
    const double v = (a11 * dot(e2, ww) - a12 * dot(e1, ww)) / det;
    w[L[0]] = 1.0;
    w[L[1]] = -(1.0 - u - v);
    w[L[2]] = -u;
    w[L[3]] = -v;
  } else {
    const d3 a0 = P[L[0]], a1 = P[L[1]], b0 = P[L[2]], b1 = P[L[3]];
    const d3 ea = a1 - a0, eb = b1 - b0, r = a0 - b0;
    const double A = dot(ea, ea), B = dot(ea, eb), C = dot(eb, eb), D = dot(ea, r), E = dot(eb, r);
    const double den = A * C - B * B;
    const double sp = (B * E - C * D) / den, tp = (A * E - B * D) / den;
    w[L[0]] = 1.0 - sp;
    w[L[1]] = sp;
    w[L[2]] = -(1.0 - tp);
    w[L[3]] = -tp;
  }
  d3 diff = mk(0, 0, 0);
  for (int a = 0; a < k; ++a) diff = diff + w[a] * P[a];
  const double d = sqrt(dot(diff, diff));
  for (int a = 0; a < 4; ++a) gam[4 * (size_t)i + a] = w[a];
  nrm[3 * (size_t)i] = diff.x / d;
  nrm[3 * (size_t)i + 1] = diff.y / d;
  nrm[3 * (size_t)i + 2] = diff.z / d;
  double p1 = 0.0;
  if (inA[i] != 0.0) p1 += sigma * barrier_b1(d, dhat);
  if (inAp[i] != 0.0) p1 += -mu[i] + sigma * barrier_b1(d, dhat + s[i]);
  lam[i] = (inA[i] != 0.0) ? -p1 : 0.0;
}

__global__ void k_node_contact_grad(int n, const int* __restrict__ rp, const int* __restrict__ col,
                                    const int* __restrict__ start, const int* __restrict__ codes,
                                    const double* __restrict__ grad_c, const uint8_t* __restrict__ fixed,
                                    double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double g[3] = {0, 0, 0};
  if (!fixed[i] && rp != nullptr) {
    for (int s = rp[i]; s < rp[i + 1]; ++s) {
      if (col[s] != i) continue;
      for (int c = start[s]; c < start[s + 1]; ++c) {
        const int code = codes[c];
        const int st = code >> 4, a = (code >> 2) & 3;
        for (int q = 0; q < 3; ++q) g[q] += grad_c[12 * (size_t)st + 3 * a + q];
      }
    }
  }
  for (int q = 0; q < 3; ++q) out[3 * (size_t)i + q] = g[q];
}

__global__ void k_velocity(int n3, const double* __restrict__ x, const double* __restrict__ xt, double inv_h,
                           double* __restrict__ v) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n3) v[j] = (x[j] - xt[j]) * inv_h;
}
__global__ void k_restore_fixed(int n, const double* __restrict__ xt, const uint8_t* __restrict__ fixed, double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && fixed[i])
    for (int c = 0; c < 3; ++c) x[3 * (size_t)i + c] = xt[3 * (size_t)i + c];
}

struct Energy {
  double L;
  int count;
  double dmin;
  double S;
  double part[5];  // elastic, inertia, barrier, AL, friction (BAL_VERBOSE=2 diagnostics)
};

// R-LS1: the line search accepts L(x + a p) <= L(x) + 8u max(S0, S1), i.e. no increase
// beyond the FP64 evaluation error of L (S = sum of the magnitudes of its terms).
constexpr double kLsRound = 8.0 * 1.1102230246251565e-16;
// R-LS1 tolerance factor; BAL_LS_ROUND overrides it (experiments only: 0 = the literal Q35 test)
inline double ls_round() {
  static const double v = getenv("BAL_LS_ROUND") ? atof(getenv("BAL_LS_ROUND")) : kLsRound;
  return v;
}
// R-FRIC1: window of the friction-anchor freeze test
constexpr int kFreezeWindow = 10;

double host_scalar(bal_ctx* c, const double* dev) {
  double v;
  CK(cudaMemcpyAsync(&v, dev, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return v;
}

// L(x) at fixed (y, sigma, A' with mu, s, friction anchors) over the swept candidate set (Q37).
Energy energy(bal_ctx* c, StepWork& w, const double* xe, const Candidates& cand, double sigma) {
  cudaStream_t st = c->st;
  const int N = c->N, T = c->T;
  const double h = c->prm.h, dhat = c->prm.dhat;
  w.esc.reserve(16);
  w.evals.reserve(std::max(N, T) + 1);
  w.cw.part.reserve(kRedBlocks);
  double* E = w.esc.ptr;
  // [0] elastic, [1] inertia, [2] barrier, [3] barrier dmin, [4] AL, [5] AL dmin, [6] friction,
  // [7] sum |AL_i|
  CK(cudaMemsetAsync(E, 0, 8 * sizeof(double), st));
  if (T > 0) {
    launch_elastic_energy(st, T, xe, c->tets.ptr, c->Dm_inv.ptr, c->vol.ptr, c->mu.ptr, c->lam.ptr,
                          c->any_arap ? c->tmodel.ptr : nullptr, w.evals.ptr);
    launch_sum(st, T, w.evals.ptr, w.cw.part.ptr, E + 0);
  }
  k_inertia_energy<<<ceil_div(N, 256), 256, 0, st>>>(N, xe, c->y.ptr, c->mass.ptr, 0.5 / (h * h), c->fixed.ptr,
                                                      w.evals.ptr);
  launch_sum(st, N, w.evals.ptr, w.cw.part.ptr, E + 1);
  const int n = constraint_set(st, w.cs_trial, cand, xe, dhat);
  barrier_energy(st, w.cw, w.cs_trial, sigma, dhat, E + 2, E + 3);
  if (w.n_ap > 0) {
    w.ap_d.reserve(w.n_ap);
    key_distances(st, w.n_ap, w.ap_keys.ptr, xe, w.ap_d.ptr);
    phi_al_energy(st, w.cw, w.n_ap, w.ap_d.ptr, w.ap_mu.ptr, w.ap_s.ptr, sigma, dhat, E + 4, E + 5, E + 7);
  } else {
    const double inf = INFINITY;
    CK(cudaMemcpyAsync(E + 5, &inf, sizeof(double), cudaMemcpyHostToDevice, st));
  }
  if (c->n_fric > 0) {
    w.evals.reserve(std::max(std::max(N, T), c->n_fric) + 1);
    launch_friction_energy(st, c->n_fric, xe, c->xt.ptr, c->fr_keys.ptr, c->fr_gam.ptr, c->fr_nrm.ptr, c->fr_lam.ptr,
                           c->prm.chi, c->prm.eps_v * h, w.evals.ptr);
    launch_sum(st, c->n_fric, w.evals.ptr, w.cw.part.ptr, E + 6);
  }
  double hv[8];
  CK(cudaMemcpyAsync(hv, E, sizeof(hv), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  c->launches += 12;
  Energy r;
  r.count = n;
  r.dmin = hv[3];
  const bool bad = !(hv[3] > 0.0) || !(hv[5] > 0.0) || !std::isfinite(hv[0]);
  const double L = hv[1] + hv[0] + hv[2] + hv[4] + hv[6];
  r.L = (bad || !std::isfinite(L)) ? INFINITY : L;
  // magnitude scale of the FP64 evaluation error of L (DESIGN.md R-LS1)
  r.S = std::fabs(hv[1]) + std::fabs(hv[0]) + std::fabs(hv[2]) + hv[7] + std::fabs(hv[6]);
  if (!std::isfinite(r.L)) r.S = INFINITY;
  r.part[0] = hv[0];
  r.part[1] = hv[1];
  r.part[2] = hv[2];
  r.part[3] = hv[4];
  r.part[4] = hv[6];
  return r;
}

double norm2(bal_ctx* c, const double* v, int n) {
  launch_dot(c->st, n, v, v, c->red.ptr, c->red.ptr + kRedBlocks + 1);
  c->launches += 2;
  return host_scalar(c, c->red.ptr + kRedBlocks + 1);
}
double dotp(bal_ctx* c, const double* a, const double* b, int n) {
  launch_dot(c->st, n, a, b, c->red.ptr, c->red.ptr + kRedBlocks + 2);
  c->launches += 2;
  return host_scalar(c, c->red.ptr + kRedBlocks + 2);
}

void proximity(bal_ctx* c, StepWork& w, const double* x) {
  broad_phase(c->st, w.cw, w.cand_prox, c->V, c->sverts.ptr, c->F, c->tris.ptr, c->E, c->edges.ptr, x, x,
              c->prm.dhat, c->fixed.ptr);
  constraint_set(c->st, w.cs_A, w.cand_prox, x, c->prm.dhat);
  c->launches += 16;
}

double min_d(bal_ctx* c, StepWork& w, const ConstraintSet& cs) {
  if (cs.n == 0) return INFINITY;
  w.cw.part.reserve(kRedBlocks);
  launch_min(c->st, cs.n, cs.d.ptr, w.cw.part.ptr, c->red.ptr + kRedBlocks + 3);
  return host_scalar(c, c->red.ptr + kRedBlocks + 3);
}

// sigma0 = max(-(g_b . g_E)/||g_b||^2, mean free mass / h^2)  (Q7)
double sigma0(bal_ctx* c, StepWork& w, const double* x) {
  cudaStream_t st = c->st;
  const int N = c->N;
  const int saved_n = c->cset.n, saved_f = c->n_fric;
  // g_E = grad (E_I + Psi): assembly with no contact stencils
  c->cset.n = 0;
  c->n_fric = 0;
  run_assembly(c, x, c->y.ptr, 1.0);
  w.gE.reserve(3 * (size_t)N);
  CK(cudaMemcpyAsync(w.gE.ptr, c->grad.ptr, 3 * (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  c->cset.n = saved_n;
  c->n_fric = saved_f;
  const double floor_ = c->mean_free_mass / (c->prm.h * c->prm.h);
  if (w.cs_A.n == 0) return floor_;
  // g_b = sum_A grad b(d; dhat): contact stencils with sigma = 1, inA = 1
  stencil_union(st, c->ks, w.cs_A.n, w.cs_A.keys.ptr, 0, nullptr, nullptr, nullptr, c->cset);
  const int ns = c->cset.n;
  c->stage_c.reserve(90 * (size_t)ns);
  c->grad_c.reserve(12 * (size_t)ns);
  c->lbar_c.reserve(ns);
  c->nodes_c.reserve(4 * (size_t)ns);
  c->dist_c.reserve(ns);
  c->dphi_c.reserve(ns);
  launch_contact(st, ns, x, c->cset.keys.ptr, c->cset.inA.ptr, c->cset.inAp.ptr, c->cset.mu.ptr, c->cset.s.ptr, 1.0,
                 c->prm.dhat, c->stage_c.ptr, c->grad_c.ptr, c->lbar_c.ptr, c->nodes_c.ptr, c->dist_c.ptr,
                 c->dphi_c.ptr);
  build_contact_pattern(st, c->cw, ns, c->nodes_c.ptr, c->fixed.ptr, N, c->stage_c.ptr);
  w.gb.reserve(3 * (size_t)N);
  const bool hc = c->cw.nslots > 0;
  k_node_contact_grad<<<ceil_div(N, 256), 256, 0, st>>>(N, hc ? c->cw.row_ptr.ptr : nullptr,
                                                         hc ? c->cw.col.ptr : nullptr, hc ? c->cw.start.ptr : nullptr,
                                                         hc ? c->cw.codes_alt.ptr : nullptr, c->grad_c.ptr,
                                                         c->fixed.ptr, w.gb.ptr);
  c->launches += 6;
  const double bb = norm2(c, w.gb.ptr, 3 * N);
  if (bb == 0.0 || !std::isfinite(bb)) return floor_;
  const double be = dotp(c, w.gb.ptr, w.gE.ptr, 3 * N);
  const double s_ls = -be / bb;
  // a non-finite least-squares value (overflowing ||g_b||^2 of extremely close pairs) falls back to
  // the floor instead of poisoning the frame (Q7 floor)
  return std::isfinite(s_ls) ? std::max(s_ls, floor_) : floor_;
}

void rebuild_aprime(bal_ctx* c, StepWork& w) {
  cudaStream_t st = c->st;
  const int n = w.cs_A.n;
  const double thr = 1e-2 * c->prm.dhat;
  int nn = 0;
  if (n > 0) {
    w.sel.reserve(n + 1);
    w.selcnt.reserve(n + 1);
    k_flag_lt<<<ceil_div(n, 256), 256, 0, st>>>(n, w.cs_A.d.ptr, thr, w.sel.ptr);
    size_t t = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, t, w.sel.ptr, w.selcnt.ptr, n + 1, st));
    w.tmp.reserve(t);
    CK(cudaMemsetAsync(w.sel.ptr + n, 0, sizeof(int), st));
    CK(cub::DeviceScan::ExclusiveSum(w.tmp.ptr, t, w.sel.ptr, w.selcnt.ptr, n + 1, st));
    CK(cudaMemcpyAsync(&nn, w.selcnt.ptr + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  w.ap_keys_new.reserve(5 * (size_t)std::max(nn, 1));
  w.ap_hi_new.reserve(std::max(nn, 1));
  w.ap_lo_new.reserve(std::max(nn, 1));
  w.ap_mu_new.reserve(std::max(nn, 1));
  w.ap_s_new.reserve(std::max(nn, 1));
  if (nn > 0) {
    k_compact_keys<<<ceil_div(n, 256), 256, 0, st>>>(n, w.sel.ptr, w.selcnt.ptr, w.cs_A.keys.ptr, w.cs_A.hi.ptr,
                                                      w.cs_A.lo.ptr, w.ap_keys_new.ptr, w.ap_hi_new.ptr,
                                                      w.ap_lo_new.ptr);
    k_carry<<<ceil_div(nn, 256), 256, 0, st>>>(nn, w.ap_hi_new.ptr, w.ap_lo_new.ptr, w.n_ap, w.ap_hi.ptr, w.ap_lo.ptr,
                                               w.ap_mu.ptr, w.ap_s.ptr, w.ap_mu_new.ptr, w.ap_s_new.ptr);
    CK(cudaGetLastError());
  }
  std::swap(w.ap_keys.ptr, w.ap_keys_new.ptr);
  std::swap(w.ap_keys.cap, w.ap_keys_new.cap);
  std::swap(w.ap_hi.ptr, w.ap_hi_new.ptr);
  std::swap(w.ap_hi.cap, w.ap_hi_new.cap);
  std::swap(w.ap_lo.ptr, w.ap_lo_new.ptr);
  std::swap(w.ap_lo.cap, w.ap_lo_new.cap);
  std::swap(w.ap_mu.ptr, w.ap_mu_new.ptr);
  std::swap(w.ap_mu.cap, w.ap_mu_new.cap);
  std::swap(w.ap_s.ptr, w.ap_s_new.ptr);
  std::swap(w.ap_s.cap, w.ap_s_new.cap);
  w.n_ap = nn;
  c->launches += 4;
}

struct StepFail : std::runtime_error {
  bal_status st;
  StepFail(bal_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// ---- Alg. 1 split into frame setup / Newton iterations / finish so callers (bench)
// can advance a frame in slices of Newton iterations; bal_step = begin + iterate(max_newton) + finish.
static int verbose_level() {
  static const int v = getenv("BAL_VERBOSE") ? std::max(1, atoi(getenv("BAL_VERBOSE"))) : 0;
  return v;
}
static bool verbose_on() { return verbose_level() > 0; }
static void vmark(bal_ctx* c, std::chrono::steady_clock::time_point& t_mark, const char* what, long long a = -1,
                  long long b = -1) {
  if (!verbose_on()) return;
  CK(cudaStreamSynchronize(c->st));
  fprintf(stderr, "[bal]   %-12s %9.2f ms  %lld %lld\n", what, ms_since(t_mark), a, b);
  t_mark = std::chrono::steady_clock::now();
}

void frame_begin(bal_ctx* c, const double* x_t, const double* v_t) {
  using clk = std::chrono::steady_clock;
  if (!c->sw) c->sw = new StepWork();
  StepWork& w = *c->sw;
  StepWork::Frame& F = w.fr;
  F = StepWork::Frame();
  F.t_start = clk::now();
  cudaStream_t st = c->st;
  const int N = c->N;
  const size_t n3 = 3 * (size_t)N;
  const bal_params& P = c->prm;
  const double h = P.h;
  c->trace.clear();
  auto t_mark = clk::now();
  for (auto* b : {&w.x, &w.xn, &w.dir, &w.rhs, &w.trial, &w.v}) b->reserve(n3);
  CK(cudaMemcpyAsync(c->xt.ptr, x_t, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  k_predictor<<<ceil_div(N, 256), 256, 0, st>>>(N, x_t, v_t, h, P.gravity[0], P.gravity[1], P.gravity[2],
                                                 c->fixed.ptr, c->y.ptr);
  CK(cudaMemcpyAsync(w.x.ptr, x_t, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  w.n_ap = 0;
  c->n_fric = 0;
  vmark(c, t_mark, "setup");
  auto t0 = clk::now();
  proximity(c, w, w.x.ptr);
  vmark(c, t_mark, "proximity", w.cand_prox.npt + w.cand_prox.nee, w.cs_A.n);
  F.dmin = min_d(c, w, w.cs_A);
  F.S.ms_collision += ms_since(t0);
  if (!(F.dmin > 0.0)) throw StepFail(BAL_E_INFEASIBLE, "bal_step: input has a surface distance <= 0");
  t0 = clk::now();
  F.sig0 = sigma0(c, w, w.x.ptr);
  vmark(c, t_mark, "sigma0");
  if (!std::isfinite(F.sig0) || !(F.sig0 > 0.0))
    throw StepFail(BAL_E_NAN, "bal_step: sigma0 is not a positive finite number");
  F.S.ms_assembly += ms_since(t0);
  F.sigma = F.sig0;
  F.dmin_prev = INFINITY;
  F.e0 = -1.0;
  F.converged = false;
  F.l = 0;
  F.active = true;
}

// Runs up to max_iters Newton iterations of the frame in progress; returns true once converged.
bool frame_iterate(bal_ctx* c, int max_iters) {
  using clk = std::chrono::steady_clock;
  if (!c->sw || !c->sw->fr.active) throw StepFail(BAL_E_INVALID_ARG, "bal_frame_iterate: no frame in progress");
  StepWork& w = *c->sw;
  StepWork::Frame& F = w.fr;
  if (F.converged) return true;
  if (F.l >= c->prm.max_newton) throw StepFail(BAL_E_NOT_CONVERGED, "bal_step: Newton iteration cap reached");
  cudaStream_t st = c->st;
  const int N = c->N;
  const bal_params& P = c->prm;
  const double dhat = P.dhat;
  const bool verbose = verbose_on();
  auto t_mark = clk::now();
  auto mark = [&](const char* what, long long a = -1, long long b = -1) { vmark(c, t_mark, what, a, b); };
  bal_step_stats& S = F.S;
  double& sigma = F.sigma;
  double& dmin = F.dmin;
  double& dmin_prev = F.dmin_prev;
  double& e0 = F.e0;
  const double sig0 = F.sig0;
  const auto t_start = F.t_start;
  const bool no_al = (P.flags & BAL_NO_AUGLAG) != 0;
  auto t0 = clk::now();
  const int l_end = std::min(P.max_newton, F.l + std::max(max_iters, 0));
  for (; F.l < l_end; ++F.l) {
    const int l = F.l;
    if (l > 0) {
      t0 = clk::now();
      proximity(c, w, w.x.ptr);
      dmin = min_d(c, w, w.cs_A);
      S.ms_collision += ms_since(t0);
    }
    S.max_constraints = std::max(S.max_constraints, w.cs_A.n);
    // A' rules (Alg. 1 lines 3-6)
    int rebuilt = 0;
    if (!no_al) {
      if (dmin > 1e-2 * dhat) {
        w.n_ap = 0;
      } else if (dmin < dmin_prev || w.n_ap == 0) {
        rebuild_aprime(c, w);
        rebuilt = 1;
      }
    }
    dmin_prev = dmin;
    S.max_aprime = std::max(S.max_aprime, w.n_ap);
    // contact stencils = A u A' (Q22)
    t0 = clk::now();
    stencil_union(st, c->ks, w.cs_A.n, w.cs_A.keys.ptr, w.n_ap, w.ap_keys.ptr, w.ap_mu.ptr, w.ap_s.ptr, c->cset);
    // friction anchors at x^l; ablation BAL_FRICTION_LAGGED: anchors of the frame's first
    // iterate kept for the whole frame (IPC's lagged, semi-implicit friction)
    const bool lagged = (P.flags & BAL_FRICTION_LAGGED) != 0;
    const bool keep = lagged ? l > 0 : F.fric_frozen;
    if (!keep) c->n_fric = 0;
    if (P.chi > 0.0 && c->cset.n > 0 && !keep) {
      const int nc = c->cset.n;
      c->fr_keys.reserve(5 * (size_t)nc);
      c->fr_gam.reserve(4 * (size_t)nc);
      c->fr_nrm.reserve(3 * (size_t)nc);
      c->fr_lam.reserve(nc);
      CK(cudaMemcpyAsync(c->fr_keys.ptr, c->cset.keys.ptr, 5 * (size_t)nc * sizeof(int), cudaMemcpyDeviceToDevice, st));
      k_friction_anchor<<<ceil_div(nc, 128), 128, 0, st>>>(nc, c->cset.keys.ptr, c->cset.inA.ptr, c->cset.inAp.ptr,
                                                           c->cset.mu.ptr, c->cset.s.ptr, sigma, dhat, w.x.ptr,
                                                           c->fr_gam.ptr, c->fr_nrm.ptr, c->fr_lam.ptr);
      c->n_fric = nc;
    }
    mark("union+fric", c->cset.n, c->n_fric);
    run_assembly(c, w.x.ptr, c->y.ptr, sigma);
    mark("assembly", c->cw.nslots);
    const double en = std::sqrt(norm2(c, c->grad.ptr, 3 * N));
    S.ms_assembly += ms_since(t0);
    if (!std::isfinite(en)) throw StepFail(BAL_E_NAN, "bal_step: ||e|| is not finite");
    if (e0 < 0) e0 = en;
    // R-FRIC1: the per-iteration anchor update is a fixed-point iteration; once
    // the best ||e|| has not halved over kFreezeWindow Newton iterations the anchors are frozen for
    // the rest of the step (IPC's semi-implicit friction, convergent)
    F.emin.push_back(F.emin.empty() ? en : std::min(F.emin.back(), en));
    if (!F.fric_frozen && !(P.flags & BAL_FRICTION_NO_FREEZE) && P.chi > 0.0 && l >= kFreezeWindow &&
        F.emin[l] > 0.5 * F.emin[l - kFreezeWindow])
      F.fric_frozen = true;
    if (e0 == 0.0) {
      F.converged = true;
      ++F.l;
      return true;
    }
    // Newton direction: A p = -e with warm start + PCG (App. B)
    launch_axpy(st, 3 * N, -2.0, c->grad.ptr, c->grad.ptr, w.rhs.ptr);  // rhs = e - 2e = -e
    t0 = clk::now();
    bal_pcg_stats ps;
    const bool warm = !(P.flags & BAL_NO_WARMSTART);
    pcg_solve(c, w.rhs.ptr, nullptr, w.dir.ptr, warm, P.pcg_rel_tol, P.pcg_stall_window, P.max_pcg, P.ws_rel_tol,
              P.ws_max_iters, &ps);
    CK(cudaStreamSynchronize(st));
    S.ms_pcg += ms_since(t0);
    mark("pcg", ps.ws_iters_max, c->h_scal->k);
    S.ws_iters += ps.ws_iters_max;
    int resumes = 0, halvings = 0, safeguard = 0;
    double alpha = 0.0, a_ccd = 1.0;
    t0 = clk::now();
    while (true) {
      // Q38 descent safeguard; a NaN dot product (PCG stopped on NaN) also takes the -D^{-1} e fallback
      if (!(dotp(c, w.dir.ptr, c->grad.ptr, 3 * N) < 0.0)) {
        launch_apply_dinv(st, N, c->dinv.ptr, c->grad.ptr, w.dir.ptr, -1.0);
        safeguard = 1;
      }
      // swept candidates x -> x + p, CCD
      launch_axpy(st, 3 * N, 1.0, w.dir.ptr, w.x.ptr, w.trial.ptr);
      broad_phase(st, w.cw, w.cand_sw, c->V, c->sverts.ptr, c->F, c->tris.ptr, c->E, c->edges.ptr, w.x.ptr,
                  w.trial.ptr, dhat, c->fixed.ptr);
      mark("swept-bp", w.cand_sw.npt, w.cand_sw.nee);
      a_ccd = ccd_step_toi(st, w.cw, w.cand_sw, w.x.ptr, w.dir.ptr, dhat,
                           (c->prm.flags & BAL_CCD_LITERAL) ? INFINITY : 1e-2);
      mark("ccd");
      alpha = std::min(1.0, a_ccd);
      const Energy E0 = energy(c, w, w.x.ptr, w.cand_sw, sigma);
      halvings = 0;
      bool ok = false;
      Energy E1{};
      while (alpha >= P.alpha_min) {
        launch_axpy(st, 3 * N, alpha, w.dir.ptr, w.x.ptr, w.trial.ptr);
        E1 = energy(c, w, w.trial.ptr, w.cand_sw, sigma);
        mark("energy", E1.count);
        if (verbose_level() >= 2)
          fprintf(stderr,
                  "[bal]     ls a=%.3e dL=%.6e  d(el)=%.3e d(in)=%.3e d(bar)=%.3e d(al)=%.3e d(fr)=%.3e dmin=%.3e n=%d\n",
                  alpha, E1.L - E0.L, E1.part[0] - E0.part[0], E1.part[1] - E0.part[1], E1.part[2] - E0.part[2],
                  E1.part[3] - E0.part[3], E1.part[4] - E0.part[4], E1.dmin, E1.count);
        // R-LS1; an infeasible trial (J <= 0, d <= 0, NaN) has L = +inf and is never accepted
        if (E1.count <= P.max_constraints && std::isfinite(E1.L) &&
            E1.L <= E0.L + ls_round() * std::max(E0.S, E1.S)) {
          ok = true;
          break;
        }
        alpha *= 0.5;
        ++halvings;
      }
      if (ok) break;
      if (resumes >= 50 || c->h_scal->k >= P.max_pcg) {
        S.ms_linesearch += ms_since(t0);
        char buf[320];
        snprintf(buf, sizeof(buf),
                 "bal_step: line search failed after %d PCG resumes (newton l=%d, alpha_ccd=%.3e, L0=%.17g, "
                 "last L1=%.17g, |C|=%d, dmin=%.3e, pcg k=%d, safeguard=%d)",
                 resumes, l, a_ccd, E0.L, E1.L, E1.count, E1.dmin, c->h_scal->k, safeguard);
        throw StepFail(BAL_E_NOT_CONVERGED, buf);
      }
      ++resumes;
      pcg_resume(c, P.pcg_resume_iters, w.dir.ptr, &ps);
    }
    S.ms_linesearch += ms_since(t0);
    S.newton_iters += 1;
    S.pcg_iters += c->h_scal->k;
    S.last_rel_grad = en / e0;
    const double rec[BAL_TRACE_FIELDS] = {(double)l, (double)w.cs_A.n, (double)w.n_ap, (double)rebuilt, dmin, sigma,
                                          (double)ps.ws_iters_max, (double)c->h_scal->k, (double)c->h_scal->stop,
                                          a_ccd, alpha, (double)halvings, (double)resumes, (double)safeguard,
                                          en / e0};
    c->trace.insert(c->trace.end(), rec, rec + BAL_TRACE_FIELDS);
    if (verbose)
      fprintf(stderr,
              "[bal] l=%d |A|=%d |A'|=%d dmin=%.3e sigma=%.3e ws=%d pcg=%d stop=%d a_ccd=%.3e a=%.3e halv=%d res=%d "
              "rel_e=%.3e cand=%d/%d t=%.1fms (coll %.1f asm %.1f pcg %.1f ls %.1f)\n",
              l, w.cs_A.n, w.n_ap, dmin, sigma, ps.ws_iters_max, c->h_scal->k, c->h_scal->stop, a_ccd, alpha, halvings,
              resumes, en / e0, w.cand_sw.npt, w.cand_sw.nee, ms_since(t_start), S.ms_collision, S.ms_assembly,
              S.ms_pcg, S.ms_linesearch);
    // x^{l+1} is in w.trial; its constraint set is w.cs_trial
    if (en <= P.newton_rel_tol * e0) {
      std::swap(w.x.ptr, w.trial.ptr);
      F.converged = true;
      ++F.l;
      return true;
    }
    if (w.n_ap > 0) {  // Alg. 1 lines 12-14
      w.ap_d.reserve(w.n_ap);
      key_distances(st, w.n_ap, w.ap_keys.ptr, w.trial.ptr, w.ap_d.ptr);
      k_al_update<<<ceil_div(w.n_ap, 256), 256, 0, st>>>(w.n_ap, w.ap_d.ptr, sigma, dhat, w.ap_mu.ptr, w.ap_s.ptr);
      c->launches += 2;
    }
    if (!no_al) {  // Alg. 1 lines 15-16
      const double dnew = min_d(c, w, w.cs_trial);
      if (dnew < 1e-2 * dhat) {
        // verbatim max (Q8); BAL_SIGMA_MIN: the capped-growth reading min(1.2 sigma, 100 sigma0)
        sigma = (P.flags & BAL_SIGMA_MIN) ? std::min(1.2 * sigma, 100.0 * sig0) : std::max(1.2 * sigma, 100.0 * sig0);
        // NEXT-1 ablation BAL_SIGMA_CAP: overall ceiling 1e8 sigma0 (SPEC S:516 reading of line 16)
        if (P.flags & BAL_SIGMA_CAP) sigma = std::min(sigma, 1e8 * sig0);
      }
    }
    std::swap(w.x.ptr, w.trial.ptr);
  }
  return F.converged;
}

void frame_finish(bal_ctx* c, double* x_next, double* v_next, bal_step_stats* stats) {
  if (!c->sw || !c->sw->fr.active) throw StepFail(BAL_E_INVALID_ARG, "bal_frame_finish: no frame in progress");
  StepWork& w = *c->sw;
  StepWork::Frame& F = w.fr;
  cudaStream_t st = c->st;
  const int N = c->N;
  const size_t n3 = 3 * (size_t)N;
  k_restore_fixed<<<ceil_div(N, 256), 256, 0, st>>>(N, c->xt.ptr, c->fixed.ptr, w.x.ptr);
  if (x_next) CK(cudaMemcpyAsync(x_next, w.x.ptr, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (v_next) k_velocity<<<ceil_div((int)n3, 256), 256, 0, st>>>((int)n3, w.x.ptr, c->xt.ptr, 1.0 / c->prm.h, v_next);
  CK(cudaStreamSynchronize(st));
  F.S.sigma0 = F.sig0;
  F.S.sigma_final = F.sigma;
  F.S.min_distance = F.dmin;
  F.S.ms_total = ms_since(F.t_start);
  if (stats) *stats = F.S;
  F.active = false;
  if (!F.converged) throw StepFail(BAL_E_NOT_CONVERGED, "bal_step: Newton iteration cap reached");
}

bal_status do_step(bal_ctx* c, const double* x_t, const double* v_t, double* x_next, double* v_next,
                   bal_step_stats* stats) {
  frame_begin(c, x_t, v_t);
  try {
    frame_iterate(c, c->prm.max_newton);
  } catch (const StepFail&) {
    // line-search failure: x_next = last accepted iterate (still intersection-free), then report it
    c->sw->fr.converged = false;
    try {
      frame_finish(c, x_next, v_next, stats);
    } catch (const StepFail&) {
    }
    throw;
  }
  frame_finish(c, x_next, v_next, stats);
  return BAL_OK;
}

template <typename F>
bal_status guard_step(bal_ctx* c, F&& f) {
  try {
    CK(cudaSetDevice(c->device));
    return f();
  } catch (const StepFail& e) {
    c->err = e.what();
    return e.st;
  } catch (const OomError& e) {
    c->err = e.what();
    return BAL_E_OOM;
  } catch (const NcclError& e) {
    c->err = e.what();
    return BAL_E_NCCL;
  } catch (const std::exception& e) {
    c->err = e.what();
    return BAL_E_CUDA;
  }
}

}  // namespace

extern "C" {

bal_status bal_step(bal_ctx* c, const double* x_t, const double* v_t, double* x_next, double* v_next,
                    bal_step_stats* stats) {
  if (!c || !x_t || !v_t || !x_next) return BAL_E_INVALID_ARG;
  return guard_step(c, [&]() { return do_step(c, x_t, v_t, x_next, v_next, stats); });
}

bal_status bal_step_host(bal_ctx* c, const double* x_t, const double* v_t, double* x_next, double* v_next,
                         bal_step_stats* stats) {
  if (!c || !x_t || !v_t || !x_next) return BAL_E_INVALID_ARG;
  return guard_step(c, [&]() {
    const size_t n3 = 3 * (size_t)c->N;
    DevBuf<double> dx, dv, dxn, dvn;
    dx.upload(x_t, n3, c->st);
    dv.upload(v_t, n3, c->st);
    dxn.reserve(n3);
    dvn.reserve(n3);
    const bal_status s = do_step(c, dx.ptr, dv.ptr, dxn.ptr, dvn.ptr, stats);
    CK(cudaMemcpyAsync(x_next, dxn.ptr, n3 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    if (v_next) CK(cudaMemcpyAsync(v_next, dvn.ptr, n3 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return s;
  });
}

bal_status bal_frame_begin(bal_ctx* c, const double* x_t, const double* v_t) {
  if (!c || !x_t || !v_t) return BAL_E_INVALID_ARG;
  return guard_step(c, [&]() {
    frame_begin(c, x_t, v_t);
    return BAL_OK;
  });
}

bal_status bal_frame_iterate(bal_ctx* c, int32_t max_iters, int32_t* converged) {
  if (!c || max_iters < 0) return BAL_E_INVALID_ARG;
  return guard_step(c, [&]() {
    const bool done = frame_iterate(c, max_iters);
    if (converged) *converged = done ? 1 : 0;
    return BAL_OK;
  });
}

bal_status bal_frame_finish(bal_ctx* c, double* x_next, double* v_next, bal_step_stats* stats) {
  if (!c) return BAL_E_INVALID_ARG;
  return guard_step(c, [&]() {
    frame_finish(c, x_next, v_next, stats);
    return BAL_OK;
  });
}

bal_status bal_frame_peek(const bal_ctx* c, bal_step_stats* stats) {
  if (!c || !stats || !c->sw || !c->sw->fr.active) return BAL_E_INVALID_ARG;
  *stats = c->sw->fr.S;
  stats->sigma0 = c->sw->fr.sig0;
  stats->sigma_final = c->sw->fr.sigma;
  stats->min_distance = c->sw->fr.dmin;
  stats->ms_total = ms_since(c->sw->fr.t_start);
  return BAL_OK;
}

bal_status bal_detect(bal_ctx* c, const double* x, int32_t* keys_out, double* d_out, int32_t max_n,
                      int32_t* n_out) {
  if (!c || !x || !n_out || max_n < 0 || (max_n > 0 && (!keys_out || !d_out))) return BAL_E_INVALID_ARG;
  return guard_step(c, [&]() {
    if (!c->sw) c->sw = new StepWork();
    StepWork& w = *c->sw;
    proximity(c, w, x);
    const int n = w.cs_A.n;
    *n_out = n;
    if (n > max_n) throw StepFail(BAL_E_INVALID_ARG, "bal_detect: more constraints than max_n");
    if (n) {
      CK(cudaMemcpyAsync(keys_out, w.cs_A.keys.ptr, 5 * (size_t)n * sizeof(int), cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(d_out, w.cs_A.d.ptr, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    }
    CK(cudaStreamSynchronize(c->st));
    return BAL_OK;
  });
}

int32_t bal_get_trace(const bal_ctx* c, double* out, int32_t max_records) {
  if (!c || !out || max_records < 0) return BAL_E_INVALID_ARG;
  const int n = (int)(c->trace.size() / BAL_TRACE_FIELDS);
  const int m = std::min(n, max_records);
  std::memcpy(out, c->trace.data(), sizeof(double) * m * BAL_TRACE_FIELDS);
  return m;
}

}  // extern "C"
