// kernels.h -- launcher declarations shared by the libbal translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"

namespace bal {

#ifndef BAL_SPMV_TILE_ROWS
#define BAL_SPMV_TILE_ROWS 16
#endif
constexpr int kSpmvTileRows = BAL_SPMV_TILE_ROWS;  // block rows per SpMV tile

// TMA-staged symmetric SpMV (k_spmv.cu): rows per tile, threads per CTA, bulk-copy ring stages
#ifndef BAL_SYM_TILE_ROWS
#define BAL_SYM_TILE_ROWS 64
#endif
#ifndef BAL_SYM_STAGES
#define BAL_SYM_STAGES 2
#endif
constexpr int kSymR = BAL_SYM_TILE_ROWS;
constexpr int kSymThreads = 256;
constexpr int kSymStages = BAL_SYM_STAGES;

constexpr int kElasticThreads = 128;
constexpr int kMaxGroups = 64;

// ---- stencils (k_stencils.cu)
void launch_elastic(cudaStream_t st, int T, const double* x, const int4* tets, const double* Dm_inv,
                    const double* vol, const double* mu, const double* lam, double* stage, double* grad,
                    double* lbar);
void launch_elastic_energy(cudaStream_t st, int T, const double* x, const int4* tets, const double* Dm_inv,
                           const double* vol, const double* mu, const double* lam, double* out);
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
struct Bsr {
  int n = 0;             // block rows
  int nnzb = 0;          // stored blocks
  const int* row_ptr = nullptr;
  const int* col = nullptr;
  const double* val = nullptr;
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
  // TMA-staged symmetric kernel (k_spmv.cu): the mirror entries of row j split by whether the
  // stored block's row i lies in j's kSymR-row tile (then the block is in shared memory: mi_loc =
  // its index within the tile's stored range) or in a later tile (gathered: mo_pos, mo_col = i).
  const int* mi_row_ptr = nullptr;             // [n+1]
  const unsigned short* mi_loc = nullptr;      // [mi_row_ptr[n]]
  const int* mo_row_ptr = nullptr;             // [n+1]
  const int* mo_pos = nullptr;                 // [mo_row_ptr[n]]
  const int* mo_col = nullptr;                 // [mo_row_ptr[n]]
  int tcap = 0, tocap = 0;                     // max stored blocks / out-of-tile mirrors of a tile
  // rows computed by the SpMV kernels: [r0, r1) (r1 < 0 = n); a rank's owned range in the
  // partitioned solve, kSymR-aligned so tiles never straddle ranks
  int r0 = 0, r1 = -1;
  BAL_HD int row_end() const { return r1 < 0 ? n : r1; }
};
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
};
constexpr double kStallRel = 1e-10;  // DESIGN.md R-PCG1
// warm-start per-group scalars
struct GrpScal {
  double rz[kMaxGroups], pq[kMaxGroups], alpha[kMaxGroups], beta[kMaxGroups], rr[kMaxGroups],
      bnorm[kMaxGroups];
  int active[kMaxGroups], iters[kMaxGroups];
  int ngroups, max_iters, any_active, pad;
  double tol;
};

void spmv_init_grids();
bool spmv_sym_usable(const Bsr& S);
void spmv_sym_prepare(const Bsr& S);
// TMA-staged symmetric SpMV; sc != nullptr fuses p^T A p and alpha (DOT).  false = not usable.
bool launch_spmv_sym(cudaStream_t st, const Bsr& S, const Bsr& C, const double* v, double* y,
                     double* partials, unsigned* counter, PcgScal* sc);
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
