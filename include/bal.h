/*
 * bal.h -- C ABI of libbal.so: the B200-native BAL inexact Newton-PCG hot path of
 * "Barrier-Augmented Lagrangian for GPU-based Elastodynamic Contact" (arXiv 2407.00046).
 *
 * Citations: P:n = PAPER.md line n (section / equation given), Qn = SURVEY.md §8(c) reading n,
 * R-xxx = DESIGN.md reading.
 *
 * General conventions (apply to every entry point):
 *  - Every function returns bal_status (0 = OK, < 0 = error) and never aborts or exits; the
 *    human-readable reason of the last failure is available from bal_last_error(ctx).
 *  - Ownership: every array passed in or out is caller-owned; no pointer is retained across
 *    calls.  bal_init copies what it needs (host arrays may be freed on return).  The library
 *    owns all of its device memory and frees it in bal_destroy.
 *  - Memory space: bal_init takes HOST arrays.  Per-step arrays are DEVICE pointers on the
 *    ctx's device (e.g. torch.Tensor.data_ptr() of a contiguous float64 CUDA tensor) unless a
 *    function says otherwise.  bal_step_host is the end-to-end variant taking HOST arrays.
 *  - Layout: positions / velocities / vectors are AoS xyz per node, float64[3*n_nodes].
 *  - Precision: FP64 throughout ("We use double precision as default").
 *  - Synchronisation: calls are stream-ordered on the ctx stream (bal_set_stream); every call
 *    returns with its results complete on that stream.
 *  - Threads: a ctx is not thread-safe; distinct ctxs are independent.
 */
#ifndef BAL_H
#define BAL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bal_ctx bal_ctx; /* opaque, owned by the library */

typedef enum {
  BAL_OK = 0,
  BAL_E_INVALID_ARG = -1,     /* NULL / out-of-range argument */
  BAL_E_BAD_MESH = -2,        /* inverted or degenerate rest tet, bad index */
  BAL_E_INFEASIBLE = -3,      /* input has a surface distance <= 0 or a tet with J <= 0 */
  BAL_E_NOT_CONVERGED = -4,   /* Newton cap or line-search failure; x_next = last accepted iterate */
  BAL_E_CONSTRAINT_BUDGET = -5,
  BAL_E_CUDA = -6,
  BAL_E_NCCL = -7,
  BAL_E_OOM = -8,
  BAL_E_NAN = -9
} bal_status;

/* Tetrahedral mesh (host arrays).  P:134-146 (§3.1): nodal positions, lumped mass from rho. */
typedef struct {
  int32_t n_nodes, n_tets;
  const double* rest_x;          /* [3*n_nodes] rest positions */
  const int32_t* tets;           /* [4*n_tets], positive orientation (det D_m > 0) */
  const uint8_t* node_fixed;     /* [n_nodes] 1 = static obstacle / Dirichlet node (App. C) */
  const int32_t* tet_material;   /* [n_tets] index into the materials array */
  int32_t n_obstacle_tris;       /* surface-only static obstacles */
  const int32_t* obstacle_tris;  /* [3*n_obstacle_tris]; every referenced node must be fixed */
} bal_mesh;

/* Neo-Hookean material (Q1: Psi = mu/2 (tr F^T F - 3) - mu ln J + lam/2 (ln J)^2). */
/* Material (Table 1 columns E, nu, rho).  model: BAL_MODEL_NEO_HOOKEAN (Q1) or BAL_MODEL_ARAP
 * (NEXT-4: Psi = mu ||F - R||_F^2, R the polar rotation; lambda unused; DESIGN.md R-ARAP). */
#define BAL_MODEL_NEO_HOOKEAN 0
#define BAL_MODEL_ARAP 1
typedef struct { double E, nu, rho; int32_t model; } bal_material;

/* Flags */
#define BAL_NO_WARMSTART 1u  /* ablation: global PCG from x0 = 0 */
#define BAL_NO_AUGLAG 2u     /* ablation: A' = {} and sigma = sigma0 (plain IPC barrier Newton) */
#define BAL_FRICTION_LAGGED 4u /* ablation (GPU only, no oracle parity): friction anchors (lambda, n, beta)
                                * of the frame's first iterate kept for the whole frame */
#define BAL_SIGMA_CAP 8u     /* NEXT-1 ablation: sigma schedule of Alg. 1 line 16 with an overall ceiling
                              * of 1e8 sigma^0 (the capped reading of Q8) */
#define BAL_SIGMA_MIN 16u    /* reading of Alg. 1 line 16 with min instead of the printed max:
                              * sigma <- min(1.2 sigma, 100 sigma^0), IPC-style capped growth */
#define BAL_FRICTION_NO_FREEZE 32u /* literal per-iteration friction anchors for the whole step: disables the
                                    * R-FRIC1 freeze (anchors frozen once min ||e|| has not halved in 10
                                    * Newton iterations) */

#define BAL_CCD_LITERAL 64u  /* literal P:468 CCD activation d_TOC < eps + dhat instead of DESIGN.md R-CCD2's
                              * eps + min(dhat, 1e-2 d_0) (ablation: shown to stall the line search) */
#define BAL_PCG_LITERAL_STALL 128u /* literal P:757 / Q15 stagnation test on the residual norm (stop when the
                                    * best ||r|| of the last window is no better than the best before it)
                                    * instead of DESIGN.md R-PCG1's CG-objective test (ablation) */

#define BAL_FP32_MATRIX 256u /* NEXT-3 ("single-precision version"): the global PCG's SpMV streams the
                              * stored static blocks rounded to FP32 (36 B instead of 72 B per block);
                              * arithmetic, vectors, contact blocks, preconditioner and warm start stay FP64 */

#define BAL_ADDITIVE_PRECOND 512u /* NEXT-1 ablation (App. A, "comparison only"): the global PCG
                                   * uses the two-level additive preconditioner M^-1 = D^-1 + sum over
                                   * 9-node aggregates of B^T (B A B^T)^-1 B (27x27 Gauss-Jordan inverses
                                   * once per Newton step; DESIGN.md R-AS1) instead of block-Jacobi D^-1;
                                   * single-GPU tile-SpMV path only (else BAL_E_INVALID_ARG) */

#define BAL_PCG_CRIT_I 1024u  /* NEXT-4 ablation, App. B criterion (i), truncated Newton: stop the global
                               * PCG at ||r|| <= min(0.5, sqrt(||grad E||)) ||grad E|| (b = -grad E) */
#define BAL_PCG_CRIT_II 2048u /* App. B criterion (ii): ||r_k|| <= u kappa(A) ||x_k|| (u = DBL_EPSILON, kappa from the
                               * assembled eigenvalues: max e_j / min e_j over free nodes, DESIGN.md R-KAPPA) */
#define BAL_PCG_CRIT_III 4096u /* App. B criterion (iii): ||r_k|| <= u kappa(A) ||b||.  (i)-(iii) replace only the
                                * relative-residual test; stagnation (R-PCG1), cap and resumes are unchanged;
                                * single-GPU tile-SpMV path only */

/* Scene / solver parameters: Table 1 columns and the constants of Alg. 1 / App. B. */
typedef struct {
  double h;              /* time step (s) */
  double gravity[3];     /* m/s^2 (Q4) */
  double dhat;           /* collision offset */
  double eps_v;          /* friction mollifier threshold */
  double chi;            /* friction coefficient */
  double newton_rel_tol; /* 1e-4, Alg. 1 line 9 */
  double pcg_rel_tol;    /* 1e-4, App. B */
  int32_t pcg_stall_window; /* 100, App. B */
  int32_t pcg_resume_iters; /* 100, App. B */
  double alpha_min;      /* 1e-9, App. B */
  double ws_rel_tol;     /* 1e-2 (Q20) */
  int32_t ws_max_iters;  /* 100 (Q20) */
  int32_t max_newton;    /* 1000 (Q13) */
  int32_t max_pcg;       /* 20000 (Q16) */
  int64_t max_constraints; /* constraint budget, P:440 (Q36) */
  uint32_t flags;        /* BAL_NO_WARMSTART | BAL_NO_AUGLAG | BAL_FRICTION_LAGGED | BAL_SIGMA_CAP | BAL_SIGMA_MIN |
                          * BAL_FRICTION_NO_FREEZE | BAL_CCD_LITERAL | BAL_PCG_LITERAL_STALL */
} bal_params;

/* Per-step statistics (Table 1 columns "avg. #iters (Newton)", "#cons"). */
typedef struct {
  int32_t newton_iters;
  int64_t pcg_iters;       /* global PCG iterations summed over Newton iterations */
  int64_t ws_iters;        /* warm-start iterations (max over groups) summed over Newton iterations */
  int32_t max_constraints; /* max |A| over Newton iterations */
  int32_t max_aprime;      /* max |A'| */
  double sigma0, sigma_final, min_distance, last_rel_grad;
  double ms_total, ms_collision, ms_assembly, ms_warmstart, ms_pcg, ms_linesearch;
} bal_step_stats;

/* Multi-GPU: one process per GPU, every call collective across the ranks.  The mesh
 * is partitioned into contiguous vertex (block-row) ranges balanced by SpMV cost and aligned to the
 * SpMV tile (bal_dist_info); each rank assembles the whole system (replicated stencils, identical
 * bits on every rank) and the global PCG / warm start are distributed: a rank computes only its
 * owned rows, receives the ghost entries of p before every SpMV (boundary-only halo of the block
 * rows its rows touch, static pattern + this Newton iteration's contact pattern) and all-reduces
 * the PCG dot products (P:381 domain-masked SpMV, P:416-423 storage; App. B decisions are taken
 * from the all-reduced scalars, so all ranks run the same iterations).  The solution slices are
 * all-gathered once per Newton iteration for the replicated line search.
 * Transport: NCCL (nccl_unique_id = the 128-byte id from bal_nccl_unique_id on rank 0, broadcast
 * by the caller, e.g. over torch.distributed) or, when host_allreduce / host_exchange are set, a
 * host transport (the library synchronises its stream and calls them on HOST buffers; tests).
 *  host_allreduce(buf, n, user): in-place elementwise sum of n doubles over the ranks; 0 = OK.
 *  host_exchange(send, send_counts, recv, recv_counts, user): counts[world] in doubles; send/recv
 *    are packed in peer order; every rank sends send[peer block] to peer and receives recv[peer
 *    block] from it; 0 = OK. */
typedef int32_t (*bal_host_allreduce_fn)(double* buf, int32_t n, void* user);
typedef int32_t (*bal_host_exchange_fn)(const double* send, const int32_t* send_counts, double* recv,
                                        const int32_t* recv_counts, void* user);
typedef struct {
  int32_t rank, world, device;
  const void* nccl_unique_id;        /* 128 bytes, or NULL with the host transport */
  bal_host_allreduce_fn host_allreduce;
  bal_host_exchange_fn host_exchange;
  void* user;
} bal_dist;

/* Writes a fresh NCCL unique id (128 bytes) to out (rank 0 calls it and broadcasts the bytes).
 * Errors: BAL_E_INVALID_ARG, BAL_E_NCCL. */
bal_status bal_nccl_unique_id(void* out128);

/* Create a context: validates the mesh, precomputes D_m^{-1}, volumes, lumped masses,
 * surface triangles / edges, the static BSR pattern and the atomic-free slot lists, and uploads
 * everything to dist->device (dist NULL = one GPU, device 0; world 1 = one GPU, no collectives).
 * With world > 1 also creates the communicator and the partition (collective over the ranks).
 * Errors: BAL_E_INVALID_ARG, BAL_E_BAD_MESH, BAL_E_CUDA, BAL_E_NCCL, BAL_E_OOM.  On error *out is
 * NULL. */
bal_status bal_init(const bal_mesh* mesh, const bal_material* materials, int32_t n_materials,
                    const bal_params* params, const bal_dist* dist, bal_ctx** out);

/* Owned block rows [*r0, *r1) of this rank and the halo of its last global PCG solve (nodes sent /
 * received per SpMV, summed over peers).  Any pointer may be NULL. */
bal_status bal_dist_info(const bal_ctx* ctx, int32_t* r0, int32_t* r1, int64_t* halo_send, int64_t* halo_recv);

/* Use `cuda_stream` (a cudaStream_t) for all subsequent work; NULL = the ctx's own stream. */
bal_status bal_set_stream(bal_ctx* ctx, void* cuda_stream);

/* One backward-Euler time step solved by Alg. 1 with the inexact
 * Newton-PCG primal solve of §4.  x_t, v_t: device [3N]; x_next: device [3N];
 * v_next: device [3N] or NULL (v_{t+1} = (x_{t+1}-x_t)/h, eq:int:x).  stats may be NULL.
 * Errors: BAL_E_INFEASIBLE (input distance <= 0), BAL_E_NOT_CONVERGED (x_next = last accepted
 * iterate, still intersection-free), BAL_E_NAN (sigma^0 or ||e^l|| not finite; x_next = last
 * accepted iterate), BAL_E_CUDA, BAL_E_OOM. */
bal_status bal_step(bal_ctx* ctx, const double* x_t, const double* v_t, double* x_next,
                    double* v_next, bal_step_stats* stats);

/* bal_step in slices (same computation, same results): bal_frame_begin does the step setup
 * (predictor y, constraint set at x_t, sigma^0; Alg. 1 lines before the loop, Q7);
 * bal_frame_iterate runs up to max_iters further inexact-Newton iterations of Alg. 1 (one l =
 * assembly + warm start + PCG + CCD line search + AL updates, Q6) and sets *converged = 1 once
 * the P:261 test passed; bal_frame_finish writes x_{t+1}, v_{t+1} (device [3N]; either may be
 * NULL) and the stats.  bal_step == begin + iterate(max_newton) + finish.  Errors as bal_step;
 * BAL_E_INVALID_ARG when no frame is in progress.  x_t, v_t are read only during begin. */
bal_status bal_frame_begin(bal_ctx* ctx, const double* x_t, const double* v_t);
bal_status bal_frame_iterate(bal_ctx* ctx, int32_t max_iters, int32_t* converged);
bal_status bal_frame_finish(bal_ctx* ctx, double* x_next, double* v_next, bal_step_stats* stats);
/* Stats of the frame in progress so far (counts and per-phase ms accumulated since begin). */
bal_status bal_frame_peek(const bal_ctx* ctx, bal_step_stats* stats);

/* End-to-end variant of bal_step: x_t, v_t, x_next, v_next are HOST arrays [3N]; the
 * host<->device copies are part of the call (used for the e2e measurement). */
bal_status bal_step_host(bal_ctx* ctx, const double* x_t, const double* v_t, double* x_next,
                         double* v_next, bal_step_stats* stats);

/* ----------------------------------------------------------------------------------------
 * Testing surface.  Same device-pointer conventions.
 * --------------------------------------------------------------------------------------*/

/* Contact state for bal_assemble: keys of the active set A and of the augmentation set A'
 * (key = [type, n0, n1, n2, n3], type 0=PP 1=PE 2=PT 3=EE, canonical node order, -1 padding;
 * Q10, Q27, Q28) with the multipliers mu and slacks s of A', penalty sigma, and the
 * friction anchors (lambda, Gamma, n) of the friction pairs (Q25, Q26).
 * All arrays are HOST arrays. */
typedef struct {
  int32_t n_active;
  const int32_t* active_keys;   /* [5*n_active] */
  int32_t n_aprime;
  const int32_t* aprime_keys;   /* [5*n_aprime] */
  const double* aprime_mu;      /* [n_aprime] */
  const double* aprime_s;       /* [n_aprime] */
  double sigma;
  int32_t n_friction;
  const int32_t* friction_keys; /* [5*n_friction] */
  const double* friction_gamma; /* [4*n_friction] signed closest-point weights */
  const double* friction_n;     /* [3*n_friction] unit normals */
  const double* friction_lambda;/* [n_friction] normal force magnitudes */
  const double* x_t;            /* HOST [3N] start-of-step positions (friction), may be NULL */
  const double* y;              /* HOST [3N] inertial predictor y = x_t + h v_t + h^2 G */
} bal_contact_state;

/* Device views of the last assembled system (valid until the next call on ctx). */
typedef struct {
  int32_t n_nodes;
  int32_t nnzb_static;          /* static (mesh-adjacency) full BSR, both triangles */
  const int32_t* static_row_ptr;/* [N+1] */
  const int32_t* static_col;    /* [nnzb_static] */
  const double* static_val;     /* [9*nnzb_static] row-major 3x3 blocks */
  int32_t nnzb_contact;         /* per-iteration contact/friction BSR, both triangles */
  const int32_t* contact_row_ptr;
  const int32_t* contact_col;
  const double* contact_val;
  const double* diag_inv;       /* [6*N] symmetric inverse of the diagonal blocks (xx xy xz yy yz zz) */
  const double* grad;           /* [3N] e = grad L, fixed entries zero */
  const double* e_node;         /* [N] assembled eigenvalue e_j */
  const int32_t* group;         /* [N] floor(log10 e_j); INT32_MIN for fixed nodes */
  int32_t n_elastic;            /* per-tet projected stencil Hessians (lower blocks) */
  const double* elastic_blocks; /* [n_tets][10][9]: blocks (a,b), a>=b, index a(a+1)/2+b */
  const double* elastic_lbar;   /* [n_tets] tr P(H)/12 */
  int32_t n_contact_stencils;
  const double* contact_blocks; /* [n][10][9] */
  const double* contact_lbar;   /* [n] */
  const int32_t* contact_stencil_nodes; /* [n][4], -1 padded */
  /* appended in round 2 (per-stencil parity of K2 / K3): the last n_friction_stencils of the
   * n_contact_stencils entries above are the friction stencils D_j, in the order of
   * bal_contact_state.friction_keys; contact_grad holds every stencil's gradient over its
   * nodes (contact: grad of phi_i(d_i); friction: grad D_j) */
  int32_t n_friction_stencils;
  const double* contact_grad;   /* [n][12] */
} bal_system_view;

/* Assemble the Newton system at x (device [3N]) for the given contact state: elastic (K1),
 * contact (K2) and friction (K3) stencils, PSD projection, atomic-free gather into BSR,
 * gradient, Lambda / e_j / groups and the block-Jacobi inverse. */
bal_status bal_assemble(bal_ctx* ctx, const double* x, const bal_contact_state* cs,
                        bal_system_view* out_view);

/* The active set A = {d < dhat} at device positions x [3N] as the GPU path builds it (Alg. 1
 * l.2; LBVH broad phase P:449-462, feature-pair distance with type resolution Q27 /
 * R-EE1, R-DUP1): keys_out HOST [5*max_n] (type, canonical nodes, -1 padded; sorted), d_out HOST
 * [max_n] the distance of each key.  *n_out = |A|.  Errors: BAL_E_INVALID_ARG (also when
 * |A| > max_n; *n_out then holds |A|). */
bal_status bal_detect(bal_ctx* ctx, const double* x, int32_t* keys_out, double* d_out, int32_t max_n,
                      int32_t* n_out);

/* Views of the system the last Newton iteration (bal_step / bal_frame_iterate) or bal_assemble
 * assembled (same fields and validity as bal_assemble's out_view).  Errors: BAL_E_INVALID_ARG. */
bal_status bal_get_system(bal_ctx* ctx, bal_system_view* out_view);

/* y = A v on the last assembled (or loaded) system.  v, y: device [3N]. */
bal_status bal_spmv(bal_ctx* ctx, const double* v, double* y);

typedef struct {
  int32_t warm_start;   /* 1 = stiffness-grouped block-Jacobi warm start (Q20), kept only if
                         * phi(x0) = x0'Ax0/2 - b'x0 < 0 = phi(0) (DESIGN.md R-WS1; else x0 = 0) */
  double rel_tol;       /* ||r|| <= rel_tol ||b|| (App. B, Q14) */
  int32_t stall_window; /* App. B stagnation window (Q15); <= 0 disables */
  int32_t max_iters;
  double ws_rel_tol;    /* Q20 */
  int32_t ws_max_iters; /* Q20 */
} bal_pcg_opts;

typedef struct {
  int32_t iters;        /* global PCG iterations */
  int32_t stop_reason;  /* 0 converged, 1 stagnated, 2 cap, 3 NaN */
  int32_t ws_iters_max; /* max warm-start iterations over groups */
  int32_t n_groups;
  double rel_residual;  /* ||r|| / ||b|| at exit */
} bal_pcg_stats;

/* Block-Jacobi PCG with the App. B policy on the last assembled (or loaded)
 * system: solves A x = rhs.  rhs, x_out device [3N]; x0 device [3N] or NULL (= 0 or the warm
 * start when opts->warm_start).  opts / stats may be NULL (defaults from bal_params). */
bal_status bal_pcg(bal_ctx* ctx, const double* rhs, const double* x0, double* x_out,
                   const bal_pcg_opts* opts, bal_pcg_stats* stats);

/* Test-only: replace the current system by a host BSR (full, both triangles, rows sorted by
 * column) so SpMV / PCG can be checked on an oracle-assembled matrix.  group may be NULL. */
typedef struct {
  int32_t n_nodes, nnzb;
  const int32_t* row_ptr; /* [N+1] */
  const int32_t* col;     /* [nnzb] */
  const double* val;      /* [9*nnzb] */
  const int32_t* group;   /* [N] or NULL */
} bal_bsr_host;
bal_status bal_load_bsr(bal_ctx* ctx, const bal_bsr_host* bsr);

/* Residual history ||r_k||, k = 0..iters, of the last global PCG solve (HOST out[max_n]);
 * returns the number of entries written (or a negative bal_status). */
int32_t bal_pcg_history(bal_ctx* ctx, double* out, int32_t max_n);
/* Decrease of the CG objective phi_0 - phi_k, k = 0..iters, of the last global PCG solve (R-PCG1's
 * stagnation measure; HOST out[max_n]); returns the number of entries written or a bal_status. */
int32_t bal_pcg_objective_history(bal_ctx* ctx, double* out, int32_t max_n);

/* Timing helper for the benchmark: run `iters` SpMV launches on the current system with CUDA
 * events on the ctx stream; returns the mean launch duration in microseconds. */
bal_status bal_bench_spmv(bal_ctx* ctx, int32_t iters, double* mean_us);

/* Decision trace of the last bal_step (SURVEY c.4): one record of BAL_TRACE_FIELDS doubles per
 * Newton iteration: l, |A|, |A'|, A'-rebuilt, min d, sigma, warm-start iters (max over groups),
 * PCG iters, PCG stop reason, alpha_CCD, alpha, halvings, resumes, descent-safeguard used,
 * ||e^l|| / ||e^0||.  `out` is a HOST array of max_records * BAL_TRACE_FIELDS doubles;
 * returns the number of records written (or a negative bal_status). */
#define BAL_TRACE_FIELDS 15
int32_t bal_get_trace(const bal_ctx* ctx, double* out, int32_t max_records);

/* SpMV instrumentation accumulated over the timed PCG SpMV launches since ctx creation (CUDA event
 * record nodes bracketing the first SpMV of every 8-iteration PCG graph batch on the ctx stream, a
 * live 1-in-8 sample): out[0] = total kernel milliseconds, out[1] = number of timed launches,
 * out[2] = algorithmic bytes (72N + 76E + 4(N+1) + 80C + 48N summed over them),
 * out[3] = bytes the configured SpMV layout must move at minimum (summed likewise).  HOST out[4]. */
bal_status bal_spmv_counters(const bal_ctx* ctx, double* out);

/* ----------------------------------------------------------------------------------------
 * Vertex-domain partition, host logic of the multi-GPU path.  HOST arrays, no
 * CUDA calls, callable without a GPU.
 * bal_partition_rows: contiguous block-row ranges [bounds[k], bounds[k+1]), k < world, balanced
 *   by row_cost[i] >= 0 (e.g. stored + mirror blocks the SpMV touches in row i); bounds[world+1].
 *   Errors: BAL_E_INVALID_ARG.
 * bal_ghost_columns: the sorted unique columns referenced by rows [r0, r1) of the CSR pattern
 *   (row_ptr[n+1], col) that lie outside [r0, r1) -- the values a rank owning [r0, r1) receives
 *   before each SpMV.  Writes min(count, cap) entries to out (may be NULL) and returns the count,
 *   or BAL_E_INVALID_ARG (< 0).
 * --------------------------------------------------------------------------------------*/
bal_status bal_partition_rows(int32_t n, const int64_t* row_cost, int32_t world, int32_t* bounds);
int32_t bal_ghost_columns(int32_t n, const int32_t* row_ptr, const int32_t* col, int32_t r0, int32_t r1,
                          int32_t* out, int32_t cap);

/* bal_halo_plan: the boundary-only halo of `rank` for the symmetric block pattern (row_ptr[n+1],
 * col; both triangles) under the partition bounds[world+1]: per peer m, the owned rows whose
 * values m needs (send_ptr[m] .. send_ptr[m+1] into send_idx, ascending) and the ghost rows owned
 * by m (recv_ptr / recv_idx, ascending).  send_ptr / recv_ptr are [world+1]; at most cap entries
 * are written to each of send_idx / recv_idx (either may be NULL).  Returns max(#send, #recv), or
 * BAL_E_INVALID_ARG (< 0).  HOST arrays, no CUDA calls.
 * bal_halo_pack / bal_halo_unpack: the pack (buf[3k+c] = v[3 idx[k]+c]) and unpack (v[3 idx[k]+c]
 * = buf[3k+c]) of the halo exchange, on HOST arrays (the device kernels use the same routine). */
int32_t bal_halo_plan(int32_t n, const int32_t* row_ptr, const int32_t* col, int32_t world, const int32_t* bounds,
                      int32_t rank, int32_t* send_ptr, int32_t* send_idx, int32_t* recv_ptr, int32_t* recv_idx,
                      int32_t cap);
bal_status bal_halo_pack(int32_t count, const int32_t* idx, const double* v, double* buf);
bal_status bal_halo_unpack(int32_t count, const int32_t* idx, const double* buf, double* v);

/* Test surface: y = A v for block rows [r0, r1) only (kSymR-aligned r0; r1 aligned or N); rows
 * outside are not written.  v, y device [3N]. */
bal_status bal_spmv_rows(bal_ctx* ctx, int32_t r0, int32_t r1, const double* v, double* y);

/* Counters of kernels launched by the library since ctx creation (bench's gpu_launches). */
int64_t bal_kernel_launches(const bal_ctx* ctx);

const char* bal_last_error(const bal_ctx* ctx);
void bal_destroy(bal_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* BAL_H */
