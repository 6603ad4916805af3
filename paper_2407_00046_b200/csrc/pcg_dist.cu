// pcg_dist.cu -- the partitioned multi-GPU solve: one process per GPU, contiguous
// vertex (block-row) ranges aligned to the SpMV tile, replicated assembly, distributed warm start
// (Q20) and global block-Jacobi PCG with the App. B policy (Q14-Q16).
// Global PCG in Chronopoulos-Gear form, per iteration: the vector update of the owned rows with the
// (r,u), (r,r) partials, halo of u (boundary rows only, grouped ncclSend/ncclRecv with the ranks
// whose rows the owned rows touch), SpMV of the owned rows with the fused (w,u) partial, ONE
// ncclAllReduce of the three sums, the scalar step (App. B stop test, alpha, beta -- identical on
// every rank because the all-reduced sums are).  The warm start keeps the textbook per-group
// recurrences.  The solution slices are all-gathered once per solve (zero-padded sum).
// A host transport (bal_dist.host_*) replaces NCCL for tests: same kernels, same data flow.
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstring>

#include "ctx.h"
#include "reduce.cuh"
#include <cmath>

namespace bal {

namespace {

constexpr int kRedHalf = 256;  // dist.red: [0, kRedHalf) local sums, [kRedHalf, 2 kRedHalf) all-reduced

#define NK(call)                                                                                            \
  do {                                                                                                      \
    ncclResult_t r_ = (call);                                                                               \
    if (r_ != ncclSuccess)                                                                                  \
      throw ::bal::NcclError(std::string("NCCL: ") + ncclGetErrorString(r_) + " at " + __FILE__ + ":" +  \
                             std::to_string(__LINE__));                                                     \
  } while (0)

inline ncclComm_t comm_of(const DistState& d) { return reinterpret_cast<ncclComm_t>(d.comm); }

// ------------------------------------------------------------------------------ kernels
__global__ void k_halo_pack(int cnt, const int32_t* __restrict__ idx, const double* __restrict__ v,
                            double* __restrict__ buf) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x)
    halo_pack_entry(k, idx, v, buf);
}
__global__ void k_halo_unpack(int cnt, const int32_t* __restrict__ idx, const double* __restrict__ buf,
                              double* __restrict__ v) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x)
    halo_unpack_entry(k, idx, buf, v);
}
// zero every entry outside the owned rows (all-gather = all-reduce of zero-padded slices, exact)
__global__ void k_zero_outside(int n3, int a3, int b3, double* __restrict__ v) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n3; j += gridDim.x * blockDim.x)
    if (j < a3 || j >= b3) v[j] = 0.0;
}

// Chronopoulos-Gear block-Jacobi PCG on the owned rows (the single-GPU recurrences of k_linalg.cu,
// oracle.linalg.pcg_cg is the parity partner): ONE all-reduce per iteration, of (r,u), (r,r) (from
// the update) and (w,u) (from the SpMV epilogue).
// init: r = b - A x0, u = M^-1 r, p = s = 0; local (r,u), (r,r), (b,b) and x0.(b + r) (R-WS1 guard)
__global__ void __launch_bounds__(kVecThreads)
k_d_cg_init(int r0, int r1, const double* __restrict__ b, const double* __restrict__ Ax0,
            const double* __restrict__ dinv, const double* __restrict__ x, double* __restrict__ r,
            double* __restrict__ u, double* __restrict__ p, double* __restrict__ s, double* partials,
            unsigned* counter, double* red_loc) {
  double loc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i = r0 + blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += gridDim.x * blockDim.x) {
    double rv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const size_t j = 3 * (size_t)i + c;
      const double bj = b[j];
      rv[c] = bj - Ax0[j];
      r[j] = rv[c];
      p[j] = 0.0;
      s[j] = 0.0;
      loc[2] += bj * bj;
      loc[3] += x[j] * (bj + rv[c]);
    }
    double u0, u1, u2;
    dinv_apply(dinv, i, rv[0], rv[1], rv[2], u0, u1, u2);
    u[3 * (size_t)i] = u0;
    u[3 * (size_t)i + 1] = u1;
    u[3 * (size_t)i + 2] = u2;
    loc[0] += rv[0] * u0 + rv[1] * u1 + rv[2] * u2;
    loc[1] += rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2];
  }
  double tot[4];
  if (last_block_reduce<4, kVecThreads>(loc, partials, counter, tot) && threadIdx.x == 0)
    for (int q = 0; q < 4; ++q) red_loc[q] = tot[q];
}
// [(r,u), (r,r)] of the last init / update, (w,u) of the SpMV epilogue and (b,b) -> the all-reduce buffer
__global__ void k_d_cg_pack(const double* red_loc, const PcgScal* lsc, double* red_glob) {
  red_glob[0] = red_loc[0];
  red_glob[1] = red_loc[1];
  red_glob[2] = lsc->pq;
  red_glob[3] = red_loc[2];
}
// after the init's all-reduce: stop-test state, then the k = 0 scalars
__global__ void k_d_cg_init_fin(PcgScal* sc, double* hist, const double* red_glob) {
  sc->bnorm = sqrt(red_glob[3]);
  sc->k = 0;
  sc->stop = -1;
  sc->done = 0;
  sc->dec = 0.0;
  sc->rz = sc->alpha = sc->beta = 0.0;
  cg_scalars(sc, hist, red_glob[0], red_glob[1], red_glob[2]);
}
// after an iteration's all-reduce: App. B stop test on ||r_k||, beta_k, alpha_k (identical on every
// rank: the all-reduced sums are)
__global__ void k_d_cg_scal(PcgScal* sc, double* hist, const double* red_glob) {
  if (sc->done) return;
  cg_scalars(sc, hist, red_glob[0], red_glob[1], red_glob[2]);
}
// update k on the owned rows: p = u + beta p, s = w + beta s (= A p), x += alpha p, r -= alpha s,
// u = M^-1 r; local (r,u), (r,r) for the next all-reduce
__global__ void __launch_bounds__(kVecThreads)
k_d_cg_update(int r0, int r1, const double* __restrict__ dinv, const double* __restrict__ w, double* __restrict__ u,
              double* __restrict__ p, double* __restrict__ s, double* __restrict__ x, double* __restrict__ r,
              double* partials, unsigned* counter, PcgScal* sc, double* red_loc) {
  if (sc->done) return;
  const double alpha = sc->alpha, beta = sc->beta;
  double loc[2] = {0.0, 0.0};
  for (int i = r0 + blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += gridDim.x * blockDim.x) {
    double rv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const size_t j = 3 * (size_t)i + c;
      const double pj = u[j] + beta * p[j];
      const double sj = w[j] + beta * s[j];
      p[j] = pj;
      s[j] = sj;
      x[j] = x[j] + alpha * pj;
      rv[c] = r[j] - alpha * sj;
      r[j] = rv[c];
    }
    double u0, u1, u2;
    dinv_apply(dinv, i, rv[0], rv[1], rv[2], u0, u1, u2);
    u[3 * (size_t)i] = u0;
    u[3 * (size_t)i + 1] = u1;
    u[3 * (size_t)i + 2] = u2;
    loc[0] += rv[0] * u0 + rv[1] * u1 + rv[2] * u2;
    loc[1] += rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2];
  }
  double tot[2];
  if (last_block_reduce<2, kVecThreads>(loc, partials, counter, tot) && threadIdx.x == 0) {
    red_loc[0] = tot[0];
    red_loc[1] = tot[1];
    sc->k = sc->k + 1;  // read by the next k_d_cg_scal only
  }
}

// ---- warm start (per-group PCG on A_GG, Q20) on the owned rows
__global__ void __launch_bounds__(kVecThreads)
k_d_ws_init(int r0, int r1, const int* __restrict__ grp, const double* __restrict__ b, const double* __restrict__ dinv,
            double* __restrict__ x, double* __restrict__ r, double* __restrict__ z, double* __restrict__ p,
            double* partials, unsigned* counter, const GrpScal* gs, double* red_loc) {
  __shared__ double bucket[(kVecThreads / 32) * kMaxGroups * 2];
  ws_zero_bucket(bucket, 2);
  const int G = gs->ngroups;
  const int stride = gridDim.x * blockDim.x;
  for (int base = r0 + blockIdx.x * blockDim.x; base < r1; base += stride) {
    const int i = base + threadIdx.x;
    int g = -1;
    double v[2] = {0.0, 0.0};
    if (i < r1) {
      g = grp[i];
      double rr[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        rr[c] = (g >= 0) ? b[3 * (size_t)i + c] : 0.0;
        r[3 * (size_t)i + c] = rr[c];
        x[3 * (size_t)i + c] = 0.0;
      }
      double z0, z1, z2;
      dinv_apply(dinv, i, rr[0], rr[1], rr[2], z0, z1, z2);
      z[3 * (size_t)i] = z0; z[3 * (size_t)i + 1] = z1; z[3 * (size_t)i + 2] = z2;
      p[3 * (size_t)i] = z0; p[3 * (size_t)i + 1] = z1; p[3 * (size_t)i + 2] = z2;
      v[0] = rr[0] * z0 + rr[1] * z1 + rr[2] * z2;
      v[1] = rr[0] * rr[0] + rr[1] * rr[1] + rr[2] * rr[2];
    }
    grp_warp_accum<2>(g, v, bucket);
  }
  double tot[2];
  if (grp_finish<2>(bucket, partials, counter, G, tot) && threadIdx.x < G) {
    red_loc[2 * threadIdx.x] = tot[0];
    red_loc[2 * threadIdx.x + 1] = tot[1];
  }
}
__global__ void k_d_ws_init_fin(GrpScal* gs, const double* red_glob) {
  const int G = gs->ngroups;
  const int g = threadIdx.x;
  if (g < G) {
    gs->rz[g] = red_glob[2 * g];
    gs->rr[g] = red_glob[2 * g + 1];
    gs->bnorm[g] = sqrt(red_glob[2 * g + 1]);
    gs->iters[g] = 0;
    const double rn = sqrt(red_glob[2 * g + 1]);
    gs->active[g] = (isfinite(rn) && !(rn <= gs->tol * gs->bnorm[g]) && gs->max_iters > 0) ? 1 : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int any = 0;
    for (int q = 0; q < G; ++q) any |= gs->active[q];
    gs->any_active = any;
  }
}
__global__ void __launch_bounds__(kVecThreads)
k_d_ws_dot(int r0, int r1, const int* __restrict__ grp, const double* __restrict__ p, const double* __restrict__ q,
           double* partials, unsigned* counter, const GrpScal* gs, double* red_loc) {
  if (!gs->any_active) return;
  __shared__ double bucket[(kVecThreads / 32) * kMaxGroups * 1];
  ws_zero_bucket(bucket, 1);
  const int G = gs->ngroups;
  const int stride = gridDim.x * blockDim.x;
  for (int base = r0 + blockIdx.x * blockDim.x; base < r1; base += stride) {
    const int i = base + threadIdx.x;
    int g = -1;
    double v[1] = {0.0};
    if (i < r1) {
      g = grp[i];
      if (g >= 0 && gs->active[g]) {
        const size_t j = 3 * (size_t)i;
        v[0] = p[j] * q[j] + p[j + 1] * q[j + 1] + p[j + 2] * q[j + 2];
      } else {
        g = -1;
      }
    }
    grp_warp_accum<1>(g, v, bucket);
  }
  double tot[1];
  if (grp_finish<1>(bucket, partials, counter, G, tot) && threadIdx.x < G) red_loc[threadIdx.x] = tot[0];
}
__global__ void __launch_bounds__(kVecThreads)
k_d_ws_update(int r0, int r1, const int* __restrict__ grp, const double* __restrict__ dinv, const double* __restrict__ p,
              const double* __restrict__ q, double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
              double* partials, unsigned* counter, const GrpScal* gs, const double* pq_glob, double* red_loc) {
  if (!gs->any_active) return;
  __shared__ double bucket[(kVecThreads / 32) * kMaxGroups * 2];
  ws_zero_bucket(bucket, 2);
  const int G = gs->ngroups;
  const int stride = gridDim.x * blockDim.x;
  for (int base = r0 + blockIdx.x * blockDim.x; base < r1; base += stride) {
    const int i = base + threadIdx.x;
    int g = -1;
    double v[2] = {0.0, 0.0};
    if (i < r1) {
      g = grp[i];
      if (g >= 0 && gs->active[g]) {
        const double alpha = gs->rz[g] / pq_glob[g];
        double rr[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const size_t j = 3 * (size_t)i + c;
          x[j] = x[j] + alpha * p[j];
          rr[c] = r[j] - alpha * q[j];
          r[j] = rr[c];
        }
        double z0, z1, z2;
        dinv_apply(dinv, i, rr[0], rr[1], rr[2], z0, z1, z2);
        z[3 * (size_t)i] = z0; z[3 * (size_t)i + 1] = z1; z[3 * (size_t)i + 2] = z2;
        v[0] = rr[0] * z0 + rr[1] * z1 + rr[2] * z2;
        v[1] = rr[0] * rr[0] + rr[1] * rr[1] + rr[2] * rr[2];
      } else {
        g = -1;
      }
    }
    grp_warp_accum<2>(g, v, bucket);
  }
  double tot[2];
  if (grp_finish<2>(bucket, partials, counter, G, tot) && threadIdx.x < G) {
    red_loc[2 * threadIdx.x] = tot[0];
    red_loc[2 * threadIdx.x + 1] = tot[1];
  }
}
__global__ void k_d_ws_fin(GrpScal* gs, const double* pq_glob, const double* rzrr_glob) {
  if (!gs->any_active) return;
  const int G = gs->ngroups;
  const int g = threadIdx.x;
  if (g < G && gs->active[g]) {
    gs->pq[g] = pq_glob[g];
    gs->alpha[g] = gs->rz[g] / pq_glob[g];
    gs->beta[g] = rzrr_glob[2 * g] / gs->rz[g];
    gs->rz[g] = rzrr_glob[2 * g];
    gs->rr[g] = rzrr_glob[2 * g + 1];
    gs->iters[g] += 1;
    const double rn = sqrt(rzrr_glob[2 * g + 1]);
    const bool stop = !isfinite(rn) || rn <= gs->tol * gs->bnorm[g] || gs->iters[g] >= gs->max_iters;
    if (stop) gs->active[g] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int any = 0;
    for (int q = 0; q < G; ++q) any |= gs->active[q];
    gs->any_active = any;
  }
}
// p = z + beta_g p on the owned rows; groups that stopped in this iteration keep p (never used again)
__global__ void k_d_ws_pupdate(int r0, int r1, const int* __restrict__ grp, const double* __restrict__ z,
                               double* __restrict__ p, const GrpScal* gs) {
  for (int i = r0 + blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += gridDim.x * blockDim.x) {
    const int g = grp[i];
    if (g >= 0 && gs->active[g]) {
      const double beta = gs->beta[g];
#pragma unroll
      for (int c = 0; c < 3; ++c) p[3 * (size_t)i + c] = z[3 * (size_t)i + c] + beta * p[3 * (size_t)i + c];
    }
  }
}

// ------------------------------------------------------------------------------ transport
void tp_allreduce(bal_ctx* c, double* dev, int n) {
  DistState& d = c->dist;
  if (d.comm) {
    NK(ncclAllReduce(dev, dev, (size_t)n, ncclDouble, ncclSum, comm_of(d), c->st));
    return;
  }
  if ((int)d.h_red.size() < n) d.h_red.resize(n);
  double* h = n <= kRedHalf ? d.h_red.data() : nullptr;
  std::vector<double> big;
  if (!h) {
    big.resize(n);
    h = big.data();
  }
  CK(cudaMemcpyAsync(h, dev, n * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (d.h_allreduce(h, n, d.user) != 0) throw CudaError("bal: host transport all-reduce failed");
  CK(cudaMemcpyAsync(dev, h, n * sizeof(double), cudaMemcpyHostToDevice, c->st));
  CK(cudaStreamSynchronize(c->st));  // h may be a local buffer
}

// halo of a [3N] vector: owned boundary rows out, ghost rows in
void tp_halo(bal_ctx* c, double* v) {
  DistState& d = c->dist;
  const int ns = (int)d.plan.send_idx.size(), nr = (int)d.plan.recv_idx.size();
  cudaStream_t st = c->st;
  if (ns > 0) k_halo_pack<<<ceil_div(ns, 256), 256, 0, st>>>(ns, d.send_idx.ptr, v, d.sbuf.ptr);
  c->launches += ns > 0;
  if (d.comm) {
    NK(ncclGroupStart());
    for (int m = 0; m < d.world; ++m) {
      const int sc = d.plan.send_ptr[m + 1] - d.plan.send_ptr[m], rc = d.plan.recv_ptr[m + 1] - d.plan.recv_ptr[m];
      if (sc > 0) NK(ncclSend(d.sbuf.ptr + 3 * (size_t)d.plan.send_ptr[m], 3 * (size_t)sc, ncclDouble, m, comm_of(d), st));
      if (rc > 0) NK(ncclRecv(d.rbuf.ptr + 3 * (size_t)d.plan.recv_ptr[m], 3 * (size_t)rc, ncclDouble, m, comm_of(d), st));
    }
    NK(ncclGroupEnd());
  } else {
    d.h_sbuf.resize(3 * (size_t)std::max(ns, 1));
    d.h_rbuf.resize(3 * (size_t)std::max(nr, 1));
    d.h_sc.assign(d.world, 0);
    d.h_rc.assign(d.world, 0);
    for (int m = 0; m < d.world; ++m) {
      d.h_sc[m] = 3 * (d.plan.send_ptr[m + 1] - d.plan.send_ptr[m]);
      d.h_rc[m] = 3 * (d.plan.recv_ptr[m + 1] - d.plan.recv_ptr[m]);
    }
    if (ns > 0) CK(cudaMemcpyAsync(d.h_sbuf.data(), d.sbuf.ptr, 3 * (size_t)ns * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (d.h_exchange(d.h_sbuf.data(), d.h_sc.data(), d.h_rbuf.data(), d.h_rc.data(), d.user) != 0)
      throw CudaError("bal: host transport exchange failed");
    if (nr > 0) CK(cudaMemcpyAsync(d.rbuf.ptr, d.h_rbuf.data(), 3 * (size_t)nr * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  if (nr > 0) k_halo_unpack<<<ceil_div(nr, 256), 256, 0, st>>>(nr, d.recv_idx.ptr, d.rbuf.ptr, v);
  c->launches += nr > 0;
  d.halo_send += ns;
  d.halo_recv += nr;
}

// all-gather of the owned slices of a [3N] vector (exact: zero-padded sum)
void tp_allgather(bal_ctx* c, double* v) {
  DistState& d = c->dist;
  const int n3 = 3 * c->N;
  k_zero_outside<<<kVecBlocks, kVecThreads, 0, c->st>>>(n3, 3 * d.r0, 3 * d.r1, v);
  c->launches += 1;
  tp_allreduce(c, v, n3);
}

// halo plan of the current system: static adjacency + this Newton iteration's contact pattern
void build_plan(bal_ctx* c) {
  DistState& d = c->dist;
  std::vector<int32_t> crp, ccol;
  const bool hc = !c->loaded_bsr && c->cw.nslots > 0;
  if (hc) {
    crp.resize(c->N + 1);
    ccol.resize(c->cw.nslots);
    CK(cudaMemcpyAsync(crp.data(), c->cw.row_ptr.ptr, crp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(ccol.data(), c->cw.col.ptr, ccol.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  halo_plan_build(c->N, d.adj_ptr.data(), d.adj_col.data(), hc ? crp.data() : nullptr, hc ? ccol.data() : nullptr,
                  d.world, d.bounds.data(), d.rank, d.plan);
  const size_t ns = d.plan.send_idx.size(), nr = d.plan.recv_idx.size();
  d.send_idx.reserve(std::max<size_t>(ns, 1));
  d.recv_idx.reserve(std::max<size_t>(nr, 1));
  if (ns) d.send_idx.upload(d.plan.send_idx.data(), ns, c->st);
  if (nr) d.recv_idx.upload(d.plan.recv_idx.data(), nr, c->st);
  d.sbuf.reserve(3 * std::max<size_t>(ns, 1));
  d.rbuf.reserve(3 * std::max<size_t>(nr, 1));
}

Bsr owned(const Bsr& S, const DistState& d) {
  Bsr b = S;
  b.ts = nullptr;  // row-range (generic) kernel on every rank: SpMV bits independent of the partition
  b.r0 = d.r0;
  b.r1 = d.r1;
  return b;
}

}  // namespace

// ------------------------------------------------------------------------------ setup
void dist_init(bal_ctx* c, const bal_dist* dd) {
  DistState& d = c->dist;
  d.rank = dd->rank;
  d.world = dd->world;
  d.h_allreduce = dd->host_allreduce;
  d.h_exchange = dd->host_exchange;
  d.user = dd->user;
  const bool host_tp = d.h_allreduce && d.h_exchange;
  if (d.world > 1 && !host_tp && !dd->nccl_unique_id)
    throw std::invalid_argument("bal_init: world > 1 needs nccl_unique_id or a host transport");
  d.active = d.world > 1 || host_tp || dd->nccl_unique_id != nullptr;
  if (!d.active) return;
  if (c->prm.flags & (BAL_ADDITIVE_PRECOND | BAL_PCG_CRIT_I | BAL_PCG_CRIT_II | BAL_PCG_CRIT_III))
    throw std::invalid_argument("bal_init: BAL_ADDITIVE_PRECOND / BAL_PCG_CRIT_* are single-GPU only");
  if (!host_tp) {
    ncclUniqueId id;
    std::memcpy(&id, dd->nccl_unique_id, sizeof(id));
    ncclComm_t comm;
    NK(ncclCommInitRank(&comm, d.world, id, d.rank));
    d.comm = comm;
  }
  // partition: contiguous block-row ranges balanced by the SpMV cost of a row (its blocks in the
  // full pattern), split points rounded to the SpMV tile so tiles never straddle ranks
  const int N = c->N;
  std::vector<int64_t> cost(N);
  for (int i = 0; i < N; ++i) cost[i] = d.adj_ptr[i + 1] - d.adj_ptr[i];
  d.bounds.assign(d.world + 1, 0);
  if (bal_partition_rows(N, cost.data(), d.world, d.bounds.data()) != BAL_OK)
    throw std::invalid_argument("bal_init: partition failed");
  for (int k = 1; k < d.world; ++k) {
    const int b = (int)(((long long)d.bounds[k] + kPartAlign / 2) / kPartAlign * kPartAlign);
    d.bounds[k] = std::max(d.bounds[k - 1], std::min(b, N));
  }
  d.bounds[d.world] = N;
  d.r0 = d.bounds[d.rank];
  d.r1 = d.bounds[d.rank + 1];
  d.red.reserve(2 * kRedHalf);
  d.lscal.reserve(1);
  CK(cudaMemsetAsync(d.lscal.ptr, 0, sizeof(PcgScal), c->st));
}

void dist_destroy(bal_ctx* c) {
  if (c->dist.comm) ncclCommDestroy(comm_of(c->dist));
  c->dist.comm = nullptr;
}

// ------------------------------------------------------------------------------ solve
namespace {

// w = A u on the owned rows after the halo of u, its (w,u) partial, one all-reduce of the packed
// scalars (4 with the init's (b,b))
void cg_spmv_reduce(bal_ctx* c, const Bsr& So, const Bsr& C, int nred) {
  DistState& d = c->dist;
  cudaStream_t st = c->st;
  tp_halo(c, c->pz.ptr);
  launch_spmv_dot(st, So, C, c->pz.ptr, c->pq.ptr, c->partials.ptr, c->counter.ptr, d.lscal.ptr);
  k_d_cg_pack<<<1, 1, 0, st>>>(d.red.ptr, d.lscal.ptr, d.red.ptr + kRedHalf);
  tp_allreduce(c, d.red.ptr + kRedHalf, nred);
  c->launches += 2;
}

void run_global(bal_ctx* c, const Bsr& So, const Bsr& C, bal_pcg_stats* stats) {
  DistState& d = c->dist;
  cudaStream_t st = c->st;
  double* red_loc = d.red.ptr;
  double* red_glob = d.red.ptr + kRedHalf;
  constexpr int kB = 8;  // iterations enqueued between polls of the device stop flag
  while (true) {
    for (int it = 0; it < kB; ++it) {
      k_d_cg_update<<<kVecBlocks, kVecThreads, 0, st>>>(d.r0, d.r1, c->dinv.ptr, c->pq.ptr, c->pz.ptr, c->pp.ptr,
                                                        c->ps.ptr, c->px.ptr, c->pr.ptr, c->partials.ptr,
                                                        c->counter.ptr, c->scal.ptr, red_loc);
      cg_spmv_reduce(c, So, C, 3);
      k_d_cg_scal<<<1, 1, 0, st>>>(c->scal.ptr, c->hist.ptr, red_glob);
      CK(cudaGetLastError());
      c->launches += 2;
    }
    CK(cudaMemcpyAsync(c->h_scal, c->scal.ptr, sizeof(PcgScal), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (c->h_scal->done) break;
  }
  if (stats) {
    double rn = 0.0;
    CK(cudaMemcpy(&rn, c->hist.ptr + c->h_scal->k, sizeof(double), cudaMemcpyDeviceToHost));
    stats->iters = c->h_scal->k;
    stats->stop_reason = c->h_scal->stop;
    stats->rel_residual = c->h_scal->bnorm > 0 ? rn / c->h_scal->bnorm : 0.0;
  }
}

}  // namespace

int pcg_solve_dist(bal_ctx* c, const double* rhs, const double* x0, double* x_out, bool warm, double tol, int window,
                   int max_iters, double ws_tol, int ws_max, bal_pcg_stats* stats) {
  DistState& d = c->dist;
  cudaStream_t st = c->st;
  const int N = c->N;
  const Bsr So = owned(c->static_bsr(), d), C = c->contact_bsr();
  if (stats) std::memset(stats, 0, sizeof(*stats));
  build_plan(c);
  const int hcap = std::max(max_iters, c->prm.max_pcg) + 8;
  if (c->hist.cap < 2 * (size_t)hcap) c->hist.reserve(2 * (size_t)hcap);
  double* red_loc = d.red.ptr;
  double* red_glob = d.red.ptr + kRedHalf;
  if (warm) {
    compact_groups(c);
    GrpScal h;
    std::memset(&h, 0, sizeof(h));
    h.ngroups = c->ngroups;
    h.max_iters = ws_max;
    h.tol = ws_tol;
    const int G = c->ngroups;
    CK(cudaMemcpyAsync(c->gscal.ptr, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    k_d_ws_init<<<kVecBlocks, kVecThreads, 0, st>>>(d.r0, d.r1, c->grp_c.ptr, rhs, c->dinv.ptr, c->px.ptr, c->pr.ptr,
                                                    c->pz.ptr, c->pp.ptr, c->partials.ptr, c->counter.ptr, c->gscal.ptr,
                                                    red_loc);
    CK(cudaMemcpyAsync(red_glob, red_loc, 2 * G * sizeof(double), cudaMemcpyDeviceToDevice, st));
    tp_allreduce(c, red_glob, 2 * G);
    k_d_ws_init_fin<<<1, kMaxGroups, 0, st>>>(c->gscal.ptr, red_glob);
    c->launches += 2;
    int done_iters = 0;
    while (done_iters < ws_max) {
      const int nb = std::min(8, ws_max - done_iters);
      for (int it = 0; it < nb; ++it) {
        tp_halo(c, c->pp.ptr);
        launch_spmv_masked(st, So, C, c->grp_c.ptr, c->pp.ptr, c->pq.ptr, c->gscal.ptr);
        k_d_ws_dot<<<kVecBlocks, kVecThreads, 0, st>>>(d.r0, d.r1, c->grp_c.ptr, c->pp.ptr, c->pq.ptr, c->partials.ptr,
                                                       c->counter.ptr, c->gscal.ptr, red_loc);
        CK(cudaMemcpyAsync(red_glob, red_loc, G * sizeof(double), cudaMemcpyDeviceToDevice, st));
        tp_allreduce(c, red_glob, G);
        k_d_ws_update<<<kVecBlocks, kVecThreads, 0, st>>>(d.r0, d.r1, c->grp_c.ptr, c->dinv.ptr, c->pp.ptr, c->pq.ptr,
                                                          c->px.ptr, c->pr.ptr, c->pz.ptr, c->partials.ptr,
                                                          c->counter.ptr, c->gscal.ptr, red_glob, red_loc);
        CK(cudaMemcpyAsync(red_glob + kMaxGroups, red_loc, 2 * G * sizeof(double), cudaMemcpyDeviceToDevice, st));
        tp_allreduce(c, red_glob + kMaxGroups, 2 * G);
        k_d_ws_fin<<<1, kMaxGroups, 0, st>>>(c->gscal.ptr, red_glob, red_glob + kMaxGroups);
        k_d_ws_pupdate<<<kVecBlocks, kVecThreads, 0, st>>>(d.r0, d.r1, c->grp_c.ptr, c->pz.ptr, c->pp.ptr, c->gscal.ptr);
        CK(cudaGetLastError());
        c->launches += 5;
      }
      done_iters += nb;
      int any = 0;
      CK(cudaMemcpyAsync(&any, &c->gscal.ptr->any_active, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
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
  } else if (x0) {
    CK(cudaMemcpyAsync(c->px.ptr, x0, 3 * (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  } else {
    CK(cudaMemsetAsync(c->px.ptr, 0, 3 * (size_t)N * sizeof(double), st));
  }
  PcgScal h;
  std::memset(&h, 0, sizeof(h));
  h.tol = tol;
  h.window = window;
  h.max_iters = max_iters;
  h.hcap = hcap;
  h.lit = (c->prm.flags & BAL_PCG_LITERAL_STALL) ? 1 : 0;
  h.pmin = INFINITY;
  h.stall_rel = stall_rel();
  CK(cudaMemcpyAsync(c->scal.ptr, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  tp_halo(c, c->px.ptr);
  launch_spmv(st, So, C, c->px.ptr, c->pq.ptr);
  k_d_cg_init<<<kVecBlocks, kVecThreads, 0, st>>>(d.r0, d.r1, rhs, c->pq.ptr, c->dinv.ptr, c->px.ptr, c->pr.ptr,
                                                  c->pz.ptr, c->pp.ptr, c->ps.ptr, c->partials.ptr, c->counter.ptr,
                                                  red_loc);
  c->launches += 2;
  c->ws_rejected = false;
  if (warm) {
    // DESIGN.md R-WS1: keep x0 only if phi(x0) = -x0'(b + r0)/2 < phi(0) = 0 (all-reduced over ranks)
    CK(cudaMemcpyAsync(red_glob, red_loc + 3, sizeof(double), cudaMemcpyDeviceToDevice, st));
    tp_allreduce(c, red_glob, 1);
    double xbr = 0.0;
    CK(cudaMemcpyAsync(&xbr, red_glob, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!(-0.5 * xbr < 0.0)) {
      CK(cudaMemsetAsync(c->px.ptr, 0, 3 * (size_t)N * sizeof(double), st));
      CK(cudaMemsetAsync(c->pq.ptr, 0, 3 * (size_t)N * sizeof(double), st));
      k_d_cg_init<<<kVecBlocks, kVecThreads, 0, st>>>(d.r0, d.r1, rhs, c->pq.ptr, c->dinv.ptr, c->px.ptr, c->pr.ptr,
                                                      c->pz.ptr, c->pp.ptr, c->ps.ptr, c->partials.ptr,
                                                      c->counter.ptr, red_loc);
      c->launches += 1;
      c->ws_rejected = true;
    }
  }
  cg_spmv_reduce(c, So, C, 4);
  k_d_cg_init_fin<<<1, 1, 0, st>>>(c->scal.ptr, c->hist.ptr, red_glob);
  CK(cudaGetLastError());
  c->launches += 1;
  CK(cudaMemcpyAsync(c->h_scal, c->scal.ptr, sizeof(PcgScal), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int ws_it = stats ? stats->ws_iters_max : 0, ng = stats ? stats->n_groups : 0;
  if (!c->h_scal->done) {
    run_global(c, So, C, stats);
  } else if (stats) {
    stats->iters = 0;
    stats->stop_reason = c->h_scal->stop;
    stats->rel_residual = c->h_scal->bnorm > 0 ? std::sqrt(c->h_scal->rr) / c->h_scal->bnorm : 0.0;
  }
  if (stats) {
    stats->ws_iters_max = ws_it;
    stats->n_groups = ng;
  }
  d.vec.reserve(3 * (size_t)N);
  CK(cudaMemcpyAsync(d.vec.ptr, c->px.ptr, 3 * (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  tp_allgather(c, d.vec.ptr);
  if (x_out) CK(cudaMemcpyAsync(x_out, d.vec.ptr, 3 * (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return c->h_scal->k;
}

// App. B resume: continue the saved distributed PCG state for `extra` more iterations
__global__ void k_d_set_resume(PcgScal* sc, int extra, int cap) {
  sc->tol = 0.0;
  sc->window = 0;
  sc->max_iters = min(sc->k + extra, cap);
  sc->done = (sc->k >= sc->max_iters) ? 1 : 0;
  sc->stop = -1;
}

void pcg_resume_dist(bal_ctx* c, int extra, double* x_out, bal_pcg_stats* stats) {
  DistState& d = c->dist;
  cudaStream_t st = c->st;
  k_d_set_resume<<<1, 1, 0, st>>>(c->scal.ptr, extra, c->prm.max_pcg);
  c->launches += 1;
  CK(cudaMemcpyAsync(c->h_scal, c->scal.ptr, sizeof(PcgScal), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const Bsr So = owned(c->static_bsr(), d), C = c->contact_bsr();
  if (!c->h_scal->done) run_global(c, So, C, stats);
  d.vec.reserve(3 * (size_t)c->N);
  CK(cudaMemcpyAsync(d.vec.ptr, c->px.ptr, 3 * (size_t)c->N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  tp_allgather(c, d.vec.ptr);
  if (x_out) CK(cudaMemcpyAsync(x_out, d.vec.ptr, 3 * (size_t)c->N * sizeof(double), cudaMemcpyDeviceToDevice, st));
}

}  // namespace bal

extern "C" {

bal_status bal_nccl_unique_id(void* out128) {
  if (!out128) return BAL_E_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return BAL_E_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return BAL_OK;
}

bal_status bal_dist_info(const bal_ctx* c, int32_t* r0, int32_t* r1, int64_t* halo_send, int64_t* halo_recv) {
  if (!c) return BAL_E_INVALID_ARG;
  if (r0) *r0 = c->dist.active ? c->dist.r0 : 0;
  if (r1) *r1 = c->dist.active ? c->dist.r1 : c->N;
  if (halo_send) *halo_send = (int64_t)c->dist.plan.send_idx.size();
  if (halo_recv) *halo_recv = (int64_t)c->dist.plan.recv_idx.size();
  return BAL_OK;
}

}  // extern "C"
