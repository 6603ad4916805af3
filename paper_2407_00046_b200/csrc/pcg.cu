// pcg.cu -- host drivers of the warm start (Q20) and the global block-Jacobi PCG with
// the App. B policy (Q14-Q16).  All scalars stay on the device; the host only polls
// the device `done` flag once per batch of kBatch iterations (kernels early-exit once done).
#include <cfloat>
#include <climits>
#include <vector>
#include <cmath>
#include <cstring>

#include "ctx.h"
#include "reduce.cuh"

namespace bal {

constexpr int kBatch = 8;
constexpr int kTimedPerBatch = 1;  // SpMV launches per batch bracketed by CUDA events

__global__ void k_group_minmax(int n, const int* __restrict__ g, int* out /*[2]*/) {
  int lo = INT_MAX, hi = INT_MIN;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = g[i];
    if (v != INT_MIN) {
      lo = min(lo, v);
      hi = max(hi, v);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
}
__global__ void k_group_compact(int n, const int* __restrict__ g, int gmin, int G, int* __restrict__ gc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int v = g[i];
  gc[i] = (v == INT_MIN) ? -1 : min(v - gmin, G - 1);
}

void compact_groups(bal_ctx* c) {
  cudaStream_t st = c->st;
  c->tmp_i.reserve(2);
  const int init[2] = {INT_MAX, INT_MIN};
  CK(cudaMemcpyAsync(c->tmp_i.ptr, init, sizeof(init), cudaMemcpyHostToDevice, st));
  k_group_minmax<<<kRedBlocks, 256, 0, st>>>(c->N, c->group.ptr, c->tmp_i.ptr);
  int mm[2];
  CK(cudaMemcpyAsync(mm, c->tmp_i.ptr, sizeof(mm), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int G = (mm[0] == INT_MAX) ? 1 : (mm[1] - mm[0] + 1);
  // more than kMaxGroups decades cannot occur for finite stiffness; the top decades are merged
  G = std::min(G, kMaxGroups);
  c->ngroups = G;
  k_group_compact<<<ceil_div(c->N, 256), 256, 0, st>>>(c->N, c->group.ptr, mm[0] == INT_MAX ? 0 : mm[0], G,
                                                       c->grp_c.ptr);
  CK(cudaGetLastError());
  c->launches += 2;
}

// NEXT-1 (App. A, R-AS1): level-2 inverses of the current system, once per solve (= once per Newton
// iteration; App. B resumes reuse them)
static void as_build(bal_ctx* c) {
  cudaStream_t st = c->st;
  const int N = c->N;
  c->as_inv.reserve((size_t)as_num_aggregates(N) * 9 * kAsAggNodes * kAsAggNodes + 1);
  const int* srp = c->loaded_bsr ? c->lb_row_ptr.ptr : c->sp.row_ptr;
  const int* scol = c->loaded_bsr ? c->lb_col.ptr : c->sp.col;
  const double* sval = c->loaded_bsr ? c->lb_val.ptr : c->sval.ptr;
  const Bsr C = c->contact_bsr();
  c->tmp_i.reserve(2);
  CK(cudaMemsetAsync(c->tmp_i.ptr, 0, sizeof(int), st));
  launch_as_build(st, N, srp, scol, sval, C.nnzb ? C.row_ptr : nullptr, C.col, C.val, c->as_inv.ptr, c->tmp_i.ptr);
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, c->tmp_i.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  c->launches += 1;
  if (bad) throw std::invalid_argument("BAL_ADDITIVE_PRECOND: an aggregate block is not positive definite");
}

static bool as_on(const bal_ctx* c) { return (c->prm.flags & BAL_ADDITIVE_PRECOND) != 0; }

// NEXT-4: App. B's alternative PCG criteria selected by flags (0 = the paper's relative residual)
static int pcg_crit(const bal_ctx* c) {
  const uint32_t f = c->prm.flags;
  return (f & BAL_PCG_CRIT_I) ? 1 : (f & BAL_PCG_CRIT_II) ? 2 : (f & BAL_PCG_CRIT_III) ? 3 : 0;
}

__global__ void k_free_minmax(int n, const double* __restrict__ e, const int* __restrict__ group,
                              double* __restrict__ part) {
  __shared__ double sh[256 / 32];
  double lo = INFINITY, hi = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (group[i] != INT_MIN) {
      lo = fmin(lo, e[i]);
      hi = fmax(hi, e[i]);
    }
  const double a = block_min<256>(lo, sh);
  const double b = -block_min<256>(-hi, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// kappa(A) estimated from the assembled eigenvalues ("approximating the condition number ...
// using our assembled eigenvalues across elasticity, collision stencils and diagonal mass matrix";
// DESIGN.md R-KAPPA): max_j e_j / min_j e_j over free nodes (Lambda is constant over a node's DOFs)
static double kappa_estimate(bal_ctx* c) {
  if (c->loaded_bsr) throw std::invalid_argument("App. B criteria (ii)/(iii) need an assembled system");
  cudaStream_t st = c->st;
  c->red.reserve(2 * kRedBlocks);
  k_free_minmax<<<kRedBlocks, 256, 0, st>>>(c->N, c->e_node.ptr, c->group.ptr, c->red.ptr);
  std::vector<double> h(2 * kRedBlocks);
  CK(cudaMemcpyAsync(h.data(), c->red.ptr, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  c->launches += 1;
  double lo = INFINITY, hi = 0.0;
  for (int b = 0; b < kRedBlocks; ++b) {
    lo = std::min(lo, h[2 * b]);
    hi = std::max(hi, h[2 * b + 1]);
  }
  return (lo > 0.0 && std::isfinite(lo)) ? hi / lo : 1.0;
}

// One batch = kBatch PCG iterations (SpMV+dot, update, p-update) + a D2H copy of the scalars and a
// completion event, captured once per solve into a CUDA graph.  Two graphs (ping-pong event sets
// and host buffers) keep one batch queued while the host inspects the previous one, so the GPU never
// idles on the host; kernels early-exit once the device `done` flag is set.
static void capture_batch(bal_ctx* c, const Bsr& S, const Bsr& C, int set, cudaGraphExec_t* out) {
  // capture on a private stream (the user's stream may be the legacy default stream, which cannot be
  // captured); the instantiated graph is then launched on the user's stream
  if (!c->cap_stream) CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  cudaStream_t st = c->cap_stream;
  const int N = c->N;
  cudaEvent_t* ev = c->ev + set * (2 * kBatch + 1);
  const bool cg = ts_usable(S);
  const int fg = cg ? 0 : pcg_fused_grid(N);  // occupancy query before the capture starts
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int it = 0; it < kBatch; ++it) {
    // CUDA events bracket the first SpMV launch of every batch (a 1-in-kBatch live sample, so the
    // event nodes do not add gaps to every iteration): the bench reports the SpMV kernel's average
    // duration inside the timed region from these (roofline achieved GB/s)
    if (cg) {
      // Chronopoulos-Gear: update k (x, r, u, p, s) then SpMV k+1 (w = A u, the iteration's one
      // grid-wide reduction, App. B stop test, alpha / beta)
      launch_cg_update(st, N, c->dinv.ptr, S.ts->pin_ptr, S.ts->part, c->pq.ptr, c->pz.ptr, c->pp.ptr, c->ps.ptr,
                       c->px.ptr, c->pr.ptr, c->upart.ptr, c->scal.ptr);
      if (as_on(c)) launch_as_apply(st, N, c->as_inv.ptr, c->pr.ptr, c->pz.ptr, c->upart.ptr, c->scal.ptr);
      if (it < kTimedPerBatch) CK(cudaEventRecordWithFlags(ev[2 * it], st, cudaEventRecordExternal));
      launch_spmv_ts_dot(st, S, C, c->pz.ptr, c->pq.ptr, S.ts->part, c->dpart.ptr, c->counter.ptr, c->scal.ptr,
                         c->upart.ptr, c->hist.ptr);
      if (it < kTimedPerBatch) CK(cudaEventRecordWithFlags(ev[2 * it + 1], st, cudaEventRecordExternal));
      continue;
    }
    if (it < kTimedPerBatch) CK(cudaEventRecordWithFlags(ev[2 * it], st, cudaEventRecordExternal));
    launch_spmv_dot(st, S, C, c->pp.ptr, c->pq.ptr, c->partials.ptr, c->counter.ptr, c->scal.ptr);
    if (it < kTimedPerBatch) CK(cudaEventRecordWithFlags(ev[2 * it + 1], st, cudaEventRecordExternal));
    if (fg > 0) {
      launch_pcg_update_fused(st, fg, N, c->dinv.ptr, c->pp.ptr, c->pq.ptr, c->px.ptr, c->pr.ptr, c->partials.ptr,
                              c->scal.ptr, c->hist.ptr);
    } else {
      launch_pcg_update(st, N, c->dinv.ptr, c->pp.ptr, c->pq.ptr, c->px.ptr, c->pr.ptr, c->pz.ptr, c->partials.ptr,
                        c->counter.ptr, c->scal.ptr, c->hist.ptr);
      launch_pcg_pupdate(st, N, c->pz.ptr, c->pp.ptr, c->scal.ptr);
    }
  }
  CK(cudaMemcpyAsync(c->h_scal + 1 + set, c->scal.ptr, sizeof(PcgScal), cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecordWithFlags(ev[2 * kBatch], st, cudaEventRecordExternal));
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(out, g, 0));
  CK(cudaGraphDestroy(g));
}

static void run_batches(bal_ctx* c, const Bsr& S, const Bsr& C, bal_pcg_stats* stats) {
  cudaStream_t st = c->st;
  if (!c->ev_ready) {
    for (int i = 0; i < 2 * (2 * kBatch + 1); ++i) CK(cudaEventCreate(&c->ev[i]));
    c->ev_ready = true;
  }
  cudaGraphExec_t ge[2];
  capture_batch(c, S, C, 0, &ge[0]);
  capture_batch(c, S, C, 1, &ge[1]);
  int k_prev = c->h_scal->k;
  CK(cudaGraphLaunch(ge[0], st));
  CK(cudaGraphLaunch(ge[1], st));
  const int per_iter = (ts_usable(S) || pcg_fused_grid(c->N) > 0) ? 2 + (as_on(c) ? 1 : 0) : 3;
  c->launches += 2 * per_iter * kBatch;
  int cur = 0;
  while (true) {
    cudaEvent_t* ev = c->ev + cur * (2 * kBatch + 1);
    CK(cudaEventSynchronize(ev[2 * kBatch]));
    const PcgScal hs = c->h_scal[1 + cur];
    // only launches that did work (iterations k_prev .. k-1) count towards the SpMV timing
    const int worked = std::min(kTimedPerBatch, hs.k - k_prev);
    for (int it = 0; it < worked; ++it) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ev[2 * it], ev[2 * it + 1]));
      c->spmv_ms += ms;
      c->spmv_count += 1;
      c->spmv_bytes_alg += c->spmv_alg_bytes();
      c->spmv_bytes_moved += c->spmv_moved_bytes();
    }
    k_prev = hs.k;
    if (hs.done) break;
    static const bool verbose = getenv("BAL_VERBOSE_PCG") != nullptr;
    if (verbose && (hs.k % 512) < kBatch)
      fprintf(stderr, "[bal-pcg] k=%d rr=%.3e bnorm=%.3e alpha=%.3e beta=%.3e\n", hs.k, std::sqrt(hs.rr), hs.bnorm,
              hs.alpha, hs.beta);
    CK(cudaGraphLaunch(ge[cur], st));  // re-queue this set behind the other in-flight batch
    c->launches += per_iter * kBatch;
    cur ^= 1;
  }
  CK(cudaStreamSynchronize(st));
  CK(cudaGraphExecDestroy(ge[0]));
  CK(cudaGraphExecDestroy(ge[1]));
  CK(cudaMemcpy(c->h_scal, c->scal.ptr, sizeof(PcgScal), cudaMemcpyDeviceToHost));
  if (stats) {
    double rn = 0.0;
    CK(cudaMemcpy(&rn, c->hist.ptr + c->h_scal->k, sizeof(double), cudaMemcpyDeviceToHost));
    stats->iters = c->h_scal->k;
    stats->stop_reason = c->h_scal->stop;
    stats->rel_residual = c->h_scal->bnorm > 0 ? rn / c->h_scal->bnorm : 0.0;
  }
}

// phi(x0) = x0'(A x0)/2 - b'x0 = -x0'(b + r0)/2 with r0 = b - A x0 (pr after the init): true when the
// warm start is not below phi(0) = 0 (R-WS1).  Two deterministic dot products and one host sync.
static bool ws_guard_rejects(bal_ctx* c, const double* rhs) {
  cudaStream_t st = c->st;
  const int n3 = 3 * c->N;
  c->red.reserve(kRedBlocks + 16);
  double* out = c->red.ptr + kRedBlocks;
  launch_dot(st, n3, c->px.ptr, rhs, c->red.ptr, out);
  launch_dot(st, n3, c->px.ptr, c->pr.ptr, c->red.ptr, out + 1);
  c->launches += 4;
  double h[2];
  CK(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double phi = -0.5 * (h[0] + h[1]);
  return !(phi < 0.0);
}

int pcg_solve(bal_ctx* c, const double* rhs, const double* x0, double* x_out, bool warm, double tol, int window,
              int max_iters, double ws_tol, int ws_max, bal_pcg_stats* stats) {
  if (c->dist.active)
    return pcg_solve_dist(c, rhs, x0, x_out, warm, tol, window, max_iters, ws_tol, ws_max, stats);
  cudaStream_t st = c->st;
  const int N = c->N;
  const Bsr S = c->static_bsr(), C = c->contact_bsr();
  if (stats) std::memset(stats, 0, sizeof(*stats));
  c->ws_rejected = false;
  // hist[0, hcap): ||r_k||; hist[hcap, 2 hcap): cumulative CG objective decrease (R-PCG1).  Sized for
  // App. B resumes up to the max_pcg cap as well.
  const int hcap = std::max(max_iters, c->prm.max_pcg) + 8;
  if (c->hist.cap < 2 * (size_t)hcap) c->hist.reserve(2 * (size_t)hcap);
  // ---------------- warm start: per-group PCG on A_GG (Q20)
  if (warm) {
    compact_groups(c);
    GrpScal h;
    std::memset(&h, 0, sizeof(h));
    h.ngroups = c->ngroups;
    h.max_iters = ws_max;
    h.tol = ws_tol;
    CK(cudaMemcpyAsync(c->gscal.ptr, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    launch_ws_init(st, N, c->grp_c.ptr, rhs, c->dinv.ptr, c->px.ptr, c->pr.ptr, c->pz.ptr, c->pp.ptr, c->partials.ptr,
                   c->counter.ptr, c->gscal.ptr);
    c->launches += 1;
    int done_iters = 0;
    while (done_iters < ws_max) {
      const int nb = std::min(kBatch, ws_max - done_iters);
      for (int it = 0; it < nb; ++it) {
        launch_spmv_masked(st, S, C, c->grp_c.ptr, c->pp.ptr, c->pq.ptr, c->gscal.ptr);
        launch_ws_dot(st, N, c->grp_c.ptr, c->pp.ptr, c->pq.ptr, c->partials.ptr, c->counter.ptr, c->gscal.ptr);
        launch_ws_update(st, N, c->grp_c.ptr, c->dinv.ptr, c->pp.ptr, c->pq.ptr, c->px.ptr, c->pr.ptr, c->pz.ptr,
                         c->partials.ptr, c->counter.ptr, c->gscal.ptr);
        launch_ws_pupdate(st, N, c->grp_c.ptr, c->pz.ptr, c->pp.ptr, c->gscal.ptr);
        c->launches += 4;
      }
      done_iters += nb;
      int any = 0;
      CK(cudaMemcpyAsync(&any, &c->gscal.ptr->any_active, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      static const bool verbose = getenv("BAL_VERBOSE_PCG") != nullptr;
      if (verbose) fprintf(stderr, "[bal-ws] it=%d G=%d any=%d\n", done_iters, c->ngroups, any);
      if (!any) break;
    }
    if (stats) {
      GrpScal g;
      CK(cudaMemcpyAsync(&g, c->gscal.ptr, sizeof(g), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      int mx = 0;
      for (int i = 0; i < g.ngroups; ++i) mx = std::max(mx, g.iters[i]);
      stats->ws_iters_max = mx;
      stats->n_groups = g.ngroups;
    }
    // x0 := warm-start result (already in px)
  } else if (x0) {
    CK(cudaMemcpyAsync(c->px.ptr, x0, 3 * (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  } else {
    CK(cudaMemsetAsync(c->px.ptr, 0, 3 * (size_t)N * sizeof(double), st));
  }
  // ---------------- global PCG from x0
  PcgScal h;
  std::memset(&h, 0, sizeof(h));
  h.tol = tol;
  h.window = window;
  h.max_iters = max_iters;
  h.hcap = hcap;
  h.lit = (c->prm.flags & BAL_PCG_LITERAL_STALL) ? 1 : 0;
  h.pmin = INFINITY;
  h.stall_rel = stall_rel();
  h.crit = pcg_crit(c);
  if (h.crit) {
    if (!ts_usable(S))
      throw std::invalid_argument("App. B criteria (i)-(iii) need the single-GPU tile-SpMV (Chronopoulos-Gear) path");
    if (h.crit >= 2) h.ukappa = DBL_EPSILON * kappa_estimate(c);
    if (h.crit == 3) h.tol = h.ukappa;
    c->last_ukappa = h.ukappa;
  }
  CK(cudaMemcpyAsync(c->scal.ptr, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  if (as_on(c)) {
    if (!ts_usable(S))
      throw std::invalid_argument("BAL_ADDITIVE_PRECOND needs the single-GPU tile-SpMV (Chronopoulos-Gear) path");
    as_build(c);
  }
  launch_spmv(st, S, C, c->px.ptr, c->pq.ptr);
  if (ts_usable(S)) {
    // single-reduction (Chronopoulos-Gear) PCG: init, then SpMV 0 (w_0 = A u_0, stop test at k = 0)
    launch_cg_init(st, N, rhs, c->pq.ptr, c->dinv.ptr, c->pr.ptr, c->pz.ptr, c->pp.ptr, c->ps.ptr, c->upart.ptr,
                   c->partials.ptr, c->counter.ptr, c->scal.ptr, c->hist.ptr, c->px.ptr);
    if (as_on(c)) launch_as_apply(st, N, c->as_inv.ptr, c->pr.ptr, c->pz.ptr, c->upart.ptr, nullptr);
    if (warm && ws_guard_rejects(c, rhs)) {
      // DESIGN.md R-WS1: the warm start is used only when it is closer to the solution than x = 0 in the
      // A-norm, phi(x0) = x0'A x0 / 2 - b'x0 < phi(0) = 0; else the solve starts from 0
      CK(cudaMemsetAsync(c->px.ptr, 0, 3 * (size_t)N * sizeof(double), st));
      CK(cudaMemsetAsync(c->pq.ptr, 0, 3 * (size_t)N * sizeof(double), st));
      launch_cg_init(st, N, rhs, c->pq.ptr, c->dinv.ptr, c->pr.ptr, c->pz.ptr, c->pp.ptr, c->ps.ptr, c->upart.ptr,
                     c->partials.ptr, c->counter.ptr, c->scal.ptr, c->hist.ptr, c->px.ptr);
      if (as_on(c)) launch_as_apply(st, N, c->as_inv.ptr, c->pr.ptr, c->pz.ptr, c->upart.ptr, nullptr);
      c->launches += 1;
      c->ws_rejected = true;
    }
    launch_spmv_ts_dot(st, S, C, c->pz.ptr, c->pq.ptr, S.ts->part, c->dpart.ptr, c->counter.ptr, c->scal.ptr,
                       c->upart.ptr, c->hist.ptr);
    c->launches += 3 + (S.ts ? 1 : 0);
  } else {
    launch_pcg_init(st, N, rhs, c->pq.ptr, c->dinv.ptr, c->pr.ptr, c->pz.ptr, c->pp.ptr, c->partials.ptr,
                    c->counter.ptr, c->scal.ptr, c->hist.ptr);
    c->launches += 2;
  }
  CK(cudaMemcpyAsync(c->h_scal, c->scal.ptr, sizeof(PcgScal), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int ws_it = stats ? stats->ws_iters_max : 0, ng = stats ? stats->n_groups : 0;
  if (!c->h_scal->done) run_batches(c, S, C, stats);
  else if (stats) {
    stats->iters = 0;
    stats->stop_reason = c->h_scal->stop;
    stats->rel_residual = c->h_scal->bnorm > 0 ? std::sqrt(c->h_scal->rr) / c->h_scal->bnorm : 0.0;
  }
  if (stats) {
    stats->ws_iters_max = ws_it;
    stats->n_groups = ng;
  }
  if (x_out && x_out != c->px.ptr)
    CK(cudaMemcpyAsync(x_out, c->px.ptr, 3 * (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return c->h_scal->k;
}

// App. B: "return to the PCG method for an additional 100 iterations" from the saved state.
__global__ void k_set_resume(PcgScal* sc, int extra, int cap) {
  sc->tol = 0.0;
  sc->crit = 0;  // App. B resume: exactly `extra` more iterations whatever the criterion
  sc->window = 0;
  sc->max_iters = min(sc->k + extra, cap);
  sc->done = (sc->k >= sc->max_iters) ? 1 : 0;
  sc->stop = -1;
}

void pcg_resume(bal_ctx* c, int extra, double* x_out, bal_pcg_stats* stats) {
  if (c->dist.active) {
    pcg_resume_dist(c, extra, x_out, stats);
    return;
  }
  cudaStream_t st = c->st;
  k_set_resume<<<1, 1, 0, st>>>(c->scal.ptr, extra, c->prm.max_pcg);
  c->launches += 1;
  const Bsr S = c->static_bsr(), C = c->contact_bsr();
  CK(cudaMemcpyAsync(c->h_scal, c->scal.ptr, sizeof(PcgScal), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (!c->h_scal->done) run_batches(c, S, C, stats);
  if (x_out && x_out != c->px.ptr)
    CK(cudaMemcpyAsync(x_out, c->px.ptr, 3 * (size_t)c->N * sizeof(double), cudaMemcpyDeviceToDevice, st));
}

}  // namespace bal
