// kernels.h -- launcher declarations shared by the libbal translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <vector>

#include "common.cuh"

namespace bal {

#ifndef BAL_SPMV_TILE_ROWS
#define BAL_SPMV_TILE_ROWS 16
#endif
constexpr int kSpmvTileRows = BAL_SPMV_TILE_ROWS;  // block rows per SpMV tile

// partitioned solve (pcg_dist.cu): rank row ranges are multiples of this (generic SpMV tiles)
constexpr int kPartAlign = 64;

// tile-symmetric SpMV (k_spmv_ts.cu): threads per CTA, TMA ring stages, max rows per tile
#ifndef BAL_TS_CONSUMERS
#define BAL_TS_CONSUMERS 256
#endif
#ifndef BAL_TS_MINB
#define BAL_TS_MINB 2
#endif
#ifndef BAL_TS_STAGES
#define BAL_TS_STAGES 2
#endif
constexpr int kTsConsumers = BAL_TS_CONSUMERS;  // consumer threads (phase 1 / phase 2)
constexpr int kTsThreads = kTsConsumers + 32;      // + one producer warp
constexpr int kTsMinBlocks = BAL_TS_MINB;  // resident CTAs per SM the tile budget is sized for
constexpr int kTsStages = BAL_TS_STAGES;
#ifndef BAL_TS_SCRATCH_BUFS
#define BAL_TS_SCRATCH_BUFS 1
#endif
constexpr int kTsScratchBufs = BAL_TS_SCRATCH_BUFS;
#ifndef BAL_TS_CONTACT_CAP
#define BAL_TS_CONTACT_CAP 384
#endif
constexpr int kTsContactCap = BAL_TS_CONTACT_CAP;  // contact blocks per tile computed block-parallel  // 2: consecutive tiles' scratch double-buffered
constexpr int kTsMaxRows = kTsConsumers;  // one consumer thread per owned row

// NEXT-1 additive preconditioner (k_additive.cu, App. A): level-2 aggregate size in nodes (27x27)
constexpr int kAsAggNodes = 9;

constexpr int kElasticThreads = 128;
constexpr int kMaxGroups = 64;

// ---- stencils (k_stencils.cu)
void launch_elastic(cudaStream_t st, int T, const double* x, const int4* tets, const double* Dm_inv,
                    const double* vol, const double* mu, const double* lam, const unsigned char* model,
                    double* stage, double* grad, double* lbar);
void launch_elastic_energy(cudaStream_t st, int T, const double* x, const int4* tets, const double* Dm_inv,
                           const double* vol, const double* mu, const double* lam, const unsigned char* model,
                           double* out);
void launch_contact(cudaStream_t st, int n, const double* x, const int* keys, const double* inA,
                    const double* inAp, const double* mu, const double* s, double sigma, double dhat,
                    double* stage, double* grad, double* lbar, int* nodes, double* dist, double* dphi);
void launch_friction(cudaStream_t st, int n, const double* x, const double* xt, const int* keys,
                     const double* gam, const double* nrm, const double* lam, double chi, double eps,
                     double* stage, double* grad, double* lbar, int* nodes);
void launch_friction_energy(cudaStream_t st, int n, const double* x, const double* xt, const int* keys,
                            const double* gam, const double* nrm, const double* lam, double chi, double eps,
                            double* out);

// ---- sparse system (k_linalg.cu)
struct TsPlan;
struct PcgScal;
struct Bsr {
  int n = 0;             // block rows
  int nnzb = 0;          // stored blocks
  const int* row_ptr = nullptr;
  const int* col = nullptr;
  const double* val = nullptr;
  const float* val32 = nullptr;  // FP32 copy of the stored blocks (BAL_FP32_MATRIX; k_spmv_ts only)
  // Symmetric storage (the paper's D + L + L^T): when m_row_ptr is set, the stored part
  // holds only the lower blocks and the diagonal (col <= row), and row i additionally applies, for
  // every j > i in m_col[m_row_ptr[i] .. m_row_ptr[i+1]), the transpose of the stored block
  // val[m_pos[.]] = A_ji.  Every off-diagonal block leaves HBM once; the mirror read is served by
  // L2 (an earlier row pulls the block, its own row streams it).  Null = every block is stored.
  const int* m_row_ptr = nullptr;  // [n+1]
  const int* m_pos = nullptr;      // [m_row_ptr[n]]
  const int* m_col = nullptr;      // [m_row_ptr[n]]
  int nmirror = 0;
  int tile_cap_s = 0;  // staged-full mode: max blocks of a kTileRows-row tile (0 = not staged)
  // tile-symmetric plan of the stored part (k_spmv_ts.cu; host-side handle, device arrays)
  const TsPlan* ts = nullptr;
  // rows computed by the SpMV kernels: [r0, r1) (r1 < 0 = n); a rank's owned range in the
  // partitioned solve, kPartAlign-aligned so tiles never straddle ranks
  int r0 = 0, r1 = -1;
  BAL_HD int row_end() const { return r1 < 0 ? n : r1; }
};
// Tile-symmetric SpMV plan (k_spmv_ts.cu): tiles of consecutive rows, per-tile metadata streamed
// with the values, partial slots of out-of-tile mirror products sorted by target row.
struct TsPlan {
  int n = 0, ntiles = 0, nslots = 0;
  // [ntiles+1] per tile: metadata offset (16 B units), first stored (lower) block, first row
  const int4* desc = nullptr;
  const unsigned char* meta = nullptr;
  const int* pin_ptr = nullptr;        // [n+1] partial slots targeting row j: [pin_ptr[j], pin_ptr[j+1])
  double* part = nullptr;              // [3 nslots] work buffer of the partials (owned by the ctx)
  int cap_nb = 0, cap_rows = 0, cap_cs = 0, cap_tp = 0;
  int val_bytes = 72;  // 72: FP64 stored blocks; 36: FP32 (BAL_FP32_MATRIX, FP64 arithmetic)
  size_t o_crp = 0;  // contact row pointers of the tile (cp.async with the out-of-tile v)
  size_t o_meta = 0, o_val = 0, o_vt = 0, o_xv = 0, stage_bytes = 0, o_scratch = 0, smem = 0;
  long long meta_bytes = 0, ncross_total = 0;
};
struct TsHost {  // host build of a TsPlan (ts_build)
  std::vector<int> tile_r0, tile_s0, pin_ptr;
  std::vector<long long> meta_off;
  std::vector<unsigned char> meta;
  int ntiles = 0, nslots = 0, cap_nb = 0, cap_rows = 0, cap_x = 0, cap_meta = 0, cap_cs = 0, cap_tp = 0;
  int val_bytes = 72;
  long long ncross_total = 0;
  size_t o_meta = 0, o_val = 0, o_vt = 0, o_xv = 0, o_crp = 0, stage_bytes = 0, o_scratch = 0, smem = 0;
};
// lower CSR (lrow[N+1], lcol: lower + diagonal blocks, ascending column) -> plan; false = unusable
bool ts_build(int N, const std::vector<int>& lrow, const std::vector<int>& lcol, int budget, int val_bytes,
              TsHost& P);
int ts_prepare(const TsPlan& P);  // grid (0 = does not fit); call outside stream capture
bool ts_usable(const Bsr& S);
// y = A v: owned rows to y, cross-tile partials to part; combine = add the partials into y
void launch_spmv_ts(cudaStream_t st, const Bsr& S, const Bsr& C, const double* v, double* y, double* part,
                    bool combine);
// w_own = A u (+ partials) with the fused single-reduction PCG epilogue (cg_scalars)
void launch_spmv_ts_dot(cudaStream_t st, const Bsr& S, const Bsr& C, const double* u, double* w, double* part,
                        double* dpart, unsigned* counter, PcgScal* sc, const double* upart, double* hist);
// App. A additive preconditioner (k_additive.cu): level-2 inverses of 9-node aggregates from the full
// static BSR + contact BSR (bad = 1 if a pivot is not positive); u += A_agg^-1 r, upart[2b] += (r, .)
int as_num_aggregates(int N);
void launch_as_build(cudaStream_t st, int N, const int* srp, const int* scol, const double* sval, const int* crp,
                     const int* ccol, const double* cval, double* inv, int* bad);
void launch_as_apply(cudaStream_t st, int N, const double* inv, const double* r, double* u, double* upart,
                     const PcgScal* sc);
// Chronopoulos-Gear PCG (k_linalg.cu): init from A x0 (complete) and the per-iteration update
void launch_cg_init(cudaStream_t st, int n, const double* b, const double* Ax0, const double* dinv, double* r,
                    double* u, double* p, double* s, double* upart, double* partials, unsigned* counter,
                    PcgScal* sc, double* hist, const double* x);
void launch_cg_update(cudaStream_t st, int n, const double* dinv, const int* pin_ptr, const double* part,
                      const double* w, double* u, double* p, double* s, double* x, double* r, double* upart,
                      PcgScal* sc);

// static-part SpMV layout: 0 = symmetric (lower + mirror index), 1 = full BSR streamed by the tiled
// kernel, 2 = full BSR staged through shared memory with cp.async.  BAL_SPMV=sym|full|staged.
inline int spmv_mode() {
  static const int m = [] {
    const char* e = getenv("BAL_SPMV");
    if (e && e[0] == 'f') return 1;
    if (e && e[0] == 's' && e[1] == 't') return 2;
    if (e && e[0] == 's') return 0;
    return getenv("BAL_SPMV_FULL") ? 1 : 0;
  }();
  return m;
}
inline bool spmv_symmetric_enabled() { return spmv_mode() == 0; }

// PCG scalars living in device memory (single group)
struct PcgScal {
  double rz, pq, alpha, beta, rr, bnorm, tol, dec;
  int k, stop, done, max_iters, window, hcap;  // hist[0..hcap) = ||r_k||, hist[hcap..) = phi_0 - phi_k
  int lit;      // BAL_PCG_LITERAL_STALL: Q15 residual-minimum stagnation test instead of R-PCG1
  double stall_rel;  // R-PCG1 threshold (kStallRel)
  double pmin;  // literal test: min ||r_j|| over j <= k - window (maintained incrementally)
  // NEXT-4 App. B alternative criteria: 0 = ||r|| <= tol ||b|| (the paper's); 1 = (i) truncated
  // Newton, tol = min(0.5, sqrt(||b||)); 2 = (ii) ||r|| <= u kappa ||x_k||; 3 = (iii) tol = u kappa
  int crit;
  double ukappa;  // u kappa(A), kappa from the assembled eigenvalues (DESIGN.md R-KAPPA)
  double xx;      // ||x_k||^2 (criterion (ii); from the update kernels' (x,x) block partials)
};
constexpr double kStallRel = 1e-10;  // DESIGN.md R-PCG1
// R-PCG1 threshold; BAL_STALL_REL overrides it (experiments)
inline double stall_rel() {
  static const double v = getenv("BAL_STALL_REL") ? atof(getenv("BAL_STALL_REL")) : kStallRel;
  return v;
}
// warm-start per-group scalars
struct GrpScal {
  double rz[kMaxGroups], pq[kMaxGroups], alpha[kMaxGroups], beta[kMaxGroups], rr[kMaxGroups],
      bnorm[kMaxGroups];
  int active[kMaxGroups], iters[kMaxGroups];
  int ngroups, max_iters, any_active, pad;
  double tol;
};

void spmv_init_grids();
void spmv_prepare(const Bsr& S);
void launch_spmv(cudaStream_t st, const Bsr& S, const Bsr& C, const double* v, double* y);
void launch_spmv_dot(cudaStream_t st, const Bsr& S, const Bsr& C, const double* v, double* y,
                     double* partials, unsigned* counter, PcgScal* sc);
void launch_pcg_init(cudaStream_t st, int n, const double* b, const double* Ax0, const double* dinv,
                     double* r, double* z, double* p, double* partials, unsigned* counter, PcgScal* sc,
                     double* hist);
void launch_pcg_update(cudaStream_t st, int n, const double* dinv, const double* p, const double* q,
                       double* x, double* r, double* z, double* partials, unsigned* counter, PcgScal* sc,
                       double* hist);
void launch_pcg_pupdate(cudaStream_t st, int n, const double* z, double* p, const PcgScal* sc);
int pcg_fused_grid(int n, int* kvariant = nullptr);
void launch_pcg_update_fused(cudaStream_t st, int grid, int n, const double* dinv, double* p, const double* q,
                             double* x, double* r, double* partials, PcgScal* sc, double* hist);

// warm start (masked SpMV + grouped scalars)
void launch_spmv_masked(cudaStream_t st, const Bsr& S, const Bsr& C, const int* grp, const double* v,
                        double* y, const GrpScal* gs);
void launch_ws_dot(cudaStream_t st, int n, const int* grp, const double* p, const double* q,
                   double* partials, unsigned* counter, GrpScal* gs);
void launch_ws_init(cudaStream_t st, int n, const int* grp, const double* b, const double* dinv, double* x,
                    double* r, double* z, double* p, double* partials, unsigned* counter, GrpScal* gs);
void launch_ws_update(cudaStream_t st, int n, const int* grp, const double* dinv, const double* p,
                      const double* q, double* x, double* r, double* z, double* partials, unsigned* counter,
                      GrpScal* gs);
void launch_ws_pupdate(cudaStream_t st, int n, const int* grp, const double* z, double* p, const GrpScal* gs);

// generic deterministic reductions
void launch_dot(cudaStream_t st, int n, const double* a, const double* b, double* partials, double* out);
void launch_sum(cudaStream_t st, int n, const double* a, double* partials, double* out);
void launch_min(cudaStream_t st, int n, const double* a, double* partials, double* out);
void launch_axpy(cudaStream_t st, int n, double alpha, const double* x, const double* y, double* out);
void launch_apply_dinv(cudaStream_t st, int nn, const double* dinv, const double* r, double* z, double scale);

}  // namespace bal
