// ctx.h -- the opaque bal_ctx: device-resident mesh, static pattern, per-iteration buffers.
#pragma once
#include <string>
#include <vector>

#include "../../include/bal.h"
#include "assemble.h"
#include "kernels.h"
#include "keys.h"
#include "halo.h"

// Device copy of a tile-symmetric SpMV plan (k_spmv_ts.cu) + its partial-slot work buffer.
struct TsDev {
  bal::DevBuf<int> pin_ptr;
  bal::DevBuf<int4> desc;
  bal::DevBuf<unsigned char> meta;
  bal::DevBuf<double> part;
  bal::TsPlan plan;
  bool ready = false;
  // lower CSR (lrow[N+1], lcol) -> plan on the device; ready = false when the kernel cannot be used
  void build(int N, const std::vector<int>& lrow, const std::vector<int>& lcol, int val_bytes, cudaStream_t st);
  void wire(bal::Bsr& b) const {
    if (ready) b.ts = &plan;
  }
};

// Partitioned solve state (pcg_dist.cu).  active = the distributed PCG path is used.
struct DistState {
  bool active = false;
  int rank = 0, world = 1, r0 = 0, r1 = 0;  // owned block rows [r0, r1)
  std::vector<int32_t> bounds;               // [world+1]
  void* comm = nullptr;                      // ncclComm_t (nullptr with the host transport)
  bal_host_allreduce_fn h_allreduce = nullptr;
  bal_host_exchange_fn h_exchange = nullptr;
  void* user = nullptr;
  std::vector<int32_t> adj_ptr, adj_col;  // static symmetric block pattern (host) for the halo plan
  bal::HaloPlan plan;
  bal::DevBuf<int> send_idx, recv_idx;
  bal::DevBuf<double> sbuf, rbuf, red, vec;  // red: [0,256) local sums, [256,512) all-reduced
  std::vector<double> h_sbuf, h_rbuf, h_red, h_vec;
  std::vector<int32_t> h_sc, h_rc;  // per-peer counts in doubles (host transport)
  bal::DevBuf<bal::PcgScal> lscal;  // sink of the owned-rows p^T A p of the SpMV epilogue
  long long halo_send = 0, halo_recv = 0;
};

struct bal_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t cap_stream = nullptr;  // CUDA-graph capture only (pcg.cu)
  cudaStream_t st = nullptr;
  bal_params prm{};
  int N = 0, T = 0;
  std::string err;
  long long launches = 0;

  // ---- mesh (device)
  bal::DevBuf<int4> tets;
  bal::DevBuf<double> Dm_inv, vol, mu, lam, mass;
  bal::DevBuf<uint8_t> fixed;
  std::vector<uint8_t> h_fixed;
  std::vector<double> h_mass;
  double mean_free_mass = 0.0;
  int n_free = 0;
  // surface
  int F = 0, E = 0, V = 0;
  bal::DevBuf<int> tris, edges, sverts;
  // ---- static pattern (device)
  bal::DevBuf<int> sp_row_ptr, sp_col, sp_slot_row, sp_diag_pos, sp_slot_ptr, sp_slot_code;
  bal::StaticPattern sp;
  bal::DevBuf<double> sval;
  bal::DevBuf<int> sp_lpos, sp_lrow, sp_lcol, sp_urow, sp_upos, sp_ucol;  // symmetric SpMV copy
  bal::DevBuf<double> lval;
  bal::DevBuf<float> lval32;  // BAL_FP32_MATRIX: FP32 copy of the stored blocks for k_spmv_ts
  bool sp_sym = false;
  TsDev sp_ts;
  bal::DevBuf<unsigned char> tmodel;  // per tet: 0 Neo-Hookean, 1 ARAP (bal_material.model)
  bool any_arap = false;
  // ---- elastic stencils
  bal::DevBuf<double> stage_e, grad_e, lbar_e;
  // ---- contact + friction stencils (friction appended after contact)
  bal::StencilSet cset;
  int n_contact = 0, n_fric = 0;
  bal::DevBuf<double> stage_c, grad_c, lbar_c, dist_c, dphi_c;
  bal::DevBuf<int> nodes_c;
  bal::DevBuf<int> fr_keys;
  bal::DevBuf<double> fr_gam, fr_nrm, fr_lam;
  bal::ContactWork cw;
  bal::KeySorter ks;
  // ---- system
  bal::DevBuf<double> grad, e_node, dinv, y, xt;
  bal::DevBuf<int> group, grp_c;
  bool loaded_bsr = false;  // test path: system injected by bal_load_bsr
  bal::DevBuf<int> lb_row_ptr, lb_col;
  bal::DevBuf<double> lb_val;
  int lb_nnzb = 0;
  // symmetric copy of the loaded system (lower + diagonal blocks, mirror index, SpMV plan)
  bal::DevBuf<int> lb_lrow, lb_lcol, lb_urow, lb_upos, lb_ucol;
  bal::DevBuf<double> lb_lval;
  bal::DevBuf<float> lb_lval32;
  int lb_nl = 0, lb_nu = 0;
  TsDev lb_ts;
  // ---- PCG
  bal::DevBuf<double> pr, pz, pp, pq, px, ps, partials, hist;
  bal::DevBuf<double> upart, dpart;  // single-reduction PCG: update-kernel and SpMV block partials
  bal::DevBuf<unsigned> counter;
  bal::DevBuf<bal::PcgScal> scal;
  bal::DevBuf<bal::GrpScal> gscal;
  bal::PcgScal* h_scal = nullptr;  // pinned
  int ngroups = 0;
  bal::DevBuf<double> as_inv;  // BAL_ADDITIVE_PRECOND: [n_agg][27][27] level-2 inverses (App. A)
  bool as_ready = false;       // as_inv holds the inverses of the current system
  bool ws_rejected = false;
  double last_ukappa = 0.0;  // u kappa of the last solve under App. B criteria (ii)/(iii)  // R-WS1: the last solve discarded its warm start
  // scratch
  bal::DevBuf<double> tmp_a, tmp_b, red;
  bal::DevBuf<int> tmp_i;

  // ---- SpMV instrumentation (CUDA events around every PCG SpMV launch)
  cudaEvent_t ev[2 * (2 * 8 + 1)] = {};  // two ping-pong sets of (2 kBatch + 1) events (pcg.cu)
  bool ev_ready = false;
  double spmv_ms = 0.0, spmv_bytes_alg = 0.0, spmv_bytes_moved = 0.0;
  long long spmv_count = 0;
  // B_alg = 72N + 76E + 4(N+1) + 80C + 48N (symmetric D/L/C layout, int32 indices)
  double spmv_alg_bytes() const {
    const double n = N;
    const double E = loaded_bsr ? 0.5 * (lb_nnzb - N) : 0.5 * (sp.nnzb - N);
    const double Cb = loaded_bsr ? 0.0 : 0.5 * (cw.nslots - cw.nrows);
    // values at the stored precision (BAL_FP32_MATRIX: 36 B per static block; contacts FP64)
    const TsDev& ts = loaded_bsr ? lb_ts : sp_ts;
    const double vb = ts.ready ? ts.plan.val_bytes : 72.0;
    return vb * n + (vb + 4.0) * E + 4.0 * (n + 1) + 80.0 * Cb + 48.0 * n;
  }
  // bytes the SpMV kernel as configured must move at minimum: the tile-symmetric kernel streams
  // lower + diagonal values (72 B), the tile metadata, v rows, out-of-tile v, y rows and partials;
  // the generic symmetric kernel streams lower + diagonal blocks (76 B with the column) and reads
  // column + mirror index (8 B) per upper slot; full mode streams every stored block
  double spmv_moved_bytes() const {
    const double n = N;
    const double cc = loaded_bsr ? 0 : cw.nslots;
    const double contact = cc > 0 ? 76.0 * cc + 4.0 * (n + 1) : 0.0;
    const TsDev& ts = loaded_bsr ? lb_ts : sp_ts;
    if (ts.ready)
      return (double)ts.plan.val_bytes * (loaded_bsr ? lb_nl : sp.nl) + (double)ts.plan.meta_bytes + 48.0 * n +
             24.0 * (double)ts.plan.ncross_total + 24.0 * ts.plan.nslots + contact;
    if (loaded_bsr) return 76.0 * lb_nnzb + 4.0 * (n + 1) + 48.0 * n;
    const double stat = sp_sym ? 76.0 * sp.nl + 8.0 * sp.nu + 8.0 * (n + 1) : 76.0 * sp.nnzb + 4.0 * (n + 1);
    return stat + contact + 48.0 * n;
  }

  DistState dist;

  // ---- time-step work (bal_step.cu), allocated on first use
  struct StepWork* sw = nullptr;
  std::vector<double> trace;  // per-Newton-iteration decision trace of the last bal_step

  bal::Bsr static_bsr() const;
  bal::Bsr contact_bsr() const;
};

void destroy_step_work(bal_ctx* c);

namespace bal {
void run_assembly(bal_ctx* c, const double* x, const double* y, double sigma);
void compact_groups(bal_ctx* c);
int pcg_solve(bal_ctx* c, const double* rhs, const double* x0, double* x_out, bool warm, double tol, int window,
              int max_iters, double ws_tol, int ws_max, bal_pcg_stats* stats);
void pcg_resume(bal_ctx* c, int extra, double* x_out, bal_pcg_stats* stats);
// partitioned solve (pcg_dist.cu)
void dist_init(bal_ctx* c, const bal_dist* d);
void dist_destroy(bal_ctx* c);
int pcg_solve_dist(bal_ctx* c, const double* rhs, const double* x0, double* x_out, bool warm, double tol, int window,
                   int max_iters, double ws_tol, int ws_max, bal_pcg_stats* stats);
void pcg_resume_dist(bal_ctx* c, int extra, double* x_out, bal_pcg_stats* stats);
}  // namespace bal
