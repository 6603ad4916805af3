// k_linalg.cu -- BSR3 SpMV, block-Jacobi PCG and the stiffness-grouped warm start
// (SURVEY §8(a) a7, a8, a9).
//
// SpMV: y = A v with A stored as a static full BSR over the mesh adjacency plus a
// per-Newton-iteration contact/friction BSR (the paper's D+L+L^T and sum C_i + C_i^T, kept as
// two row-owned parts so no atomics are needed).  Sub-warp of kSL lanes per block row: the row's
// 9*nnz doubles are contiguous, so lanes stream them perfectly coalesced; each lane accumulates
// into the 3 row components and the sub-warp reduces with shuffles.
// PCG (App. B): textbook preconditioned CG (same recurrences as the
// oracle) with M = blockdiag(D_j)^{-1} stored symmetric (6 doubles / node).  Reductions are
// deterministic: fixed grid, per-block partials, the last block (atomic ticket) reduces them in
// a fixed order and computes alpha / beta / stop flags on the device -- no host round trip.
// Warm start (Q20): per-group PCG on A_GG, masked SpMV (cross-group blocks
// skipped), per-group scalars in one GrpScal, group-wise deterministic warp-match reductions.
#include <algorithm>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "reduce.cuh"

namespace bal {

constexpr int kSL = 16;        // lanes per block row
#ifndef BAL_SPMV_THREADS
#define BAL_SPMV_THREADS 128
#endif
#ifndef BAL_SPMV_MINBLOCKS
#define BAL_SPMV_MINBLOCKS 16
#endif
#ifndef BAL_SPMV_TILE_CAP
#define BAL_SPMV_TILE_CAP 320
#endif
constexpr int kSpmvThreads = BAL_SPMV_THREADS;
constexpr int kSpmvMinBlocks = BAL_SPMV_MINBLOCKS;  // 16 x 128 threads resident per SM: independent tile pipelines
constexpr int kTileRows = kSpmvTileRows;  // block rows per SpMV tile
// persistent grid: exactly the resident CTAs, so the grid-stride sweep visits rows in increasing
// order wave by wave (the mirror-block L2 reuse above depends on it)
template <bool DOT, bool MASK>
__global__ void k_spmv(Bsr S, Bsr C, const int* __restrict__ grp, const double* __restrict__ v,
                       double* __restrict__ y, double* partials, unsigned* counter, PcgScal* sc, const GrpScal* gs);
template <bool DOT, bool MASK>
static int spmv_grid(const Bsr& S) {
  const int n = S.row_end() - (S.r0 / kTileRows) * kTileRows;
  static int per_sm = 0;
  if (per_sm == 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv<DOT, MASK>, kSpmvThreads, 0));
    per_sm = std::max(per_sm, 1);
  }
  return std::max(1, std::min(per_sm * num_sms(), ceil_div((long long)n, kTileRows)));
}

// Tiled, flattened SpMV.  A CTA owns a tile of kTileRows consecutive block rows and walks the
// tile's blocks from up to three lists -- the stored static blocks (lower + diagonal in symmetric
// mode, all blocks otherwise), the mirror entries of the static part (transposes of stored blocks
// A_ji, j > i) and the stored contact blocks -- as ONE flat sequence, so the dependent loads
// (row pointers -> column / mirror index -> values and v) cost three latency levels per tile, not
// per row.  Stage 1: row pointers of the tile (and groups when masked) to shared memory.  Stage 2:
// per block, its column and value-block index.  Stage 3: per (block, component row r) item, the
// 3-term product of row r (stored) or column r (mirror) with v at the block's column -> shared
// memory.  Stage 4: thread (row, r) sums its blocks in fixed order (list 0, 1, 2; ascending) --
// bitwise deterministic, atomic-free.  Stored blocks are streamed with L2 evict_first, mirror
// blocks read with evict_last (the earlier row pulls the block, its own row streams it); the grid
// is persistent (the resident CTAs) and sweeps tiles in increasing order, so both reads of a
// block fall within one L2 lifetime.
constexpr int kTileCap = BAL_SPMV_TILE_CAP;  // blocks staged per chunk

BAL_D unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
BAL_D unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
BAL_D double ld_hint(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

struct SpmvSmem {
  int rp[3][kTileRows + 1];
  int rgrp[kTileRows];
  int bcol[kTileCap];
  int bblk[kTileCap];
  unsigned char blist[kTileCap];
  double contrib[kTileCap][3];
};

template <bool DOT, bool MASK>
__global__ void __launch_bounds__(kSpmvThreads, kSpmvMinBlocks)
k_spmv(Bsr S, Bsr C, const int* __restrict__ grp, const double* __restrict__ v, double* __restrict__ y,
       double* partials, unsigned* counter, PcgScal* sc, const GrpScal* gs) {
  if (DOT && sc->done) return;
  __shared__ SpmvSmem sm;
  const int n = S.n;
  const int tid = threadIdx.x;
  const unsigned long long pol_first = policy_evict_first(), pol_last = policy_evict_last();
  const int ntiles = (S.row_end() + kTileRows - 1) / kTileRows;
  const int* crp = C.nnzb > 0 ? C.row_ptr : nullptr;
  double dacc = 0.0;
  for (int tile = S.r0 / kTileRows + blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int r0 = tile * kTileRows;
    const int R = min(kTileRows, S.row_end() - r0);
    // ---- stage 1: row pointers (3 lists) and row groups
    for (int t = tid; t < 3 * (kTileRows + 1); t += blockDim.x) {
      const int L = t / (kTileRows + 1), k = t - L * (kTileRows + 1);
      const int* rp = L == 0 ? S.row_ptr : (L == 1 ? S.m_row_ptr : crp);
      sm.rp[L][k] = (rp && k <= R) ? __ldg(rp + r0 + k) : 0;
    }
    if (MASK && tid < R) {
      const int g = grp[r0 + tid];
      sm.rgrp[tid] = (g >= 0 && gs->active[g]) ? g : -1;
    }
    __syncthreads();
    const int n0 = sm.rp[0][R] - sm.rp[0][0];
    const int n1 = S.m_row_ptr ? sm.rp[1][R] - sm.rp[1][0] : 0;
    const int n2 = crp ? sm.rp[2][R] - sm.rp[2][0] : 0;
    const int nt = n0 + n1 + n2;
    // thread (row, r) accumulator, persistent across chunks
    const int my_row = tid / 3, my_r = tid - 3 * (tid / 3);
    const bool reducer = tid < 3 * R;
    double acc = 0.0;
    for (int c0 = 0; c0 < nt; c0 += kTileCap) {
      const int nb = min(kTileCap, nt - c0);
      // ---- stage 2: column and value-block index of every block of the chunk
      for (int b = tid; b < nb; b += blockDim.x) {
        const int g = c0 + b;
        int col, blk, L;
        if (g < n0) {
          blk = sm.rp[0][0] + g;
          col = __ldg(S.col + blk);
          L = 0;
        } else if (g < n0 + n1) {
          const int m = sm.rp[1][0] + (g - n0);
          blk = __ldg(S.m_pos + m);
          col = __ldg(S.m_col + m);
          L = 1;
        } else {
          blk = sm.rp[2][0] + (g - n0 - n1);
          col = __ldg(C.col + blk);
          L = 2;
        }
        sm.bcol[b] = col;
        sm.bblk[b] = blk;
        sm.blist[b] = (unsigned char)L;
      }
      __syncthreads();
      // ---- stage 3: item (b, r): row r (stored) / column r (mirror) of the block times v[col]
      const int ni = 3 * nb;
#pragma unroll 4
      for (int k = tid; k < ni; k += blockDim.x) {
        const int b = k / 3, r = k - 3 * (k / 3);
        const int L = sm.blist[b];
        const int col = sm.bcol[b];
        const bool tr = L == 1;
        const double* __restrict__ pv = (L == 2 ? C.val : S.val) + 9 * (size_t)sm.bblk[b] + (tr ? r : 3 * r);
        const int st = tr ? 3 : 1;
        const unsigned long long pol = tr ? pol_last : pol_first;
        const double* __restrict__ vc = v + 3 * (size_t)col;
        const double a0 = ld_hint(pv, pol), a1 = ld_hint(pv + st, pol), a2 = ld_hint(pv + 2 * st, pol);
        const double x0 = __ldg(vc), x1 = __ldg(vc + 1), x2 = __ldg(vc + 2);
        sm.contrib[b][r] = fma(a2, x2, fma(a1, x1, a0 * x0));
      }
      __syncthreads();
      // ---- stage 4: fixed-order row sums (list 0, then 1, then 2; ascending)
      if (reducer) {
        const int gr = MASK ? sm.rgrp[my_row] : 0;
        int off = 0;
#pragma unroll
        for (int L = 0; L < 3; ++L) {
          const int nL = L == 0 ? n0 : (L == 1 ? n1 : n2);
          if (nL > 0) {
            const int lo = max(off + sm.rp[L][my_row] - sm.rp[L][0], c0);
            const int hi = min(off + sm.rp[L][my_row + 1] - sm.rp[L][0], c0 + nb);
            for (int g = lo; g < hi; ++g) {
              if (MASK && __ldg(grp + sm.bcol[g - c0]) != gr) continue;
              acc += sm.contrib[g - c0][my_r];
            }
          }
          off += nL;
        }
      }
      __syncthreads();
    }
    if (reducer) {
      const int row = r0 + my_row;
      const bool valid = !MASK || sm.rgrp[my_row] >= 0;
      if (valid) {
        y[3 * (size_t)row + my_r] = acc;
        if (DOT) dacc += v[3 * (size_t)row + my_r] * acc;
      }
    }
    __syncthreads();  // sm.rp / rgrp are rewritten by the next tile
  }
  if (DOT) {
    __shared__ double sh[kSpmvThreads / 32];
    __shared__ bool last;
    const double bs = block_sum<kSpmvThreads>(dacc, sh);
    if (threadIdx.x == 0) {
      partials[blockIdx.x] = bs;
      __threadfence();
      last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
      __threadfence();
      double t = 0.0;
      for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t += partials[i];
      t = block_sum<kSpmvThreads>(t, sh);
      if (threadIdx.x == 0) {
        sc->pq = t;
        sc->alpha = sc->rz / t;
        *counter = 0u;
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// k_spmv_sf ("staged full"): full static BSR (both triangles stored), each 16-row tile's blocks and
// columns are one contiguous range, copied to shared memory with 16-byte cp.async (L2 evict_first)
// one tile ahead while the CTA computes the previous tile from shared memory; only v (L2-resident)
// and the few contact blocks are gathered.  More bytes than the symmetric layout, but a pure
// streaming access pattern (no mirror gathers, no strided LSU traffic on the values).
BAL_D void cp_async16(void* dst, const void* src, unsigned long long pol) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "l"(pol));
}
BAL_D void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
BAL_D void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

struct SfLayout {
  size_t o_sc, stride, o_contrib, o_rp, total;
  BAL_HD void init(int cap) {
    auto up16 = [](size_t x) { return (x + 15) & ~(size_t)15; };
    o_sc = up16((size_t)(cap * 9 + 4) * 8);
    stride = up16(o_sc + (size_t)(cap + 8) * 4);
    o_contrib = 2 * stride;
    o_rp = up16(o_contrib + (size_t)cap * 24);
    total = up16(o_rp + 2 * (kTileRows + 1) * 4);
  }
};

BAL_D int stage_range(unsigned char* dst, const void* src, long long lo, long long hi, int esz,
                      unsigned long long pol) {
  if (hi <= lo) return 0;
  const size_t b0 = (size_t)lo * esz, b1 = (size_t)hi * esz;
  const size_t a0 = b0 & ~(size_t)15;
  const int nch = (int)((b1 - a0 + 15) >> 4);
  for (int c = threadIdx.x; c < nch; c += blockDim.x)
    cp_async16(dst + 16 * (size_t)c, (const unsigned char*)src + a0 + 16 * (size_t)c, pol);
  return (int)((b0 - a0) / esz);
}

template <bool DOT>
__global__ void __launch_bounds__(kSpmvThreads)
k_spmv_sf(Bsr S, Bsr C, const double* __restrict__ v, double* __restrict__ y, double* partials, unsigned* counter,
          PcgScal* sc) {
  if (DOT && sc->done) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  SfLayout Lo;
  Lo.init(S.tile_cap_s);
  int(*rp)[kTileRows + 1] = reinterpret_cast<int(*)[kTileRows + 1]>(smraw + Lo.o_rp);
  double(*contrib)[3] = reinterpret_cast<double(*)[3]>(smraw + Lo.o_contrib);
  const int n = S.n;
  const int tid = threadIdx.x;
  const unsigned long long pol_first = policy_evict_first();
  const int ntiles = (n + kTileRows - 1) / kTileRows;
  const int* crp = C.nnzb > 0 ? C.row_ptr : nullptr;
  int offv[2] = {0, 0}, offc[2] = {0, 0};
  auto load_rp = [&](int tile, int buf) {
    const int r0 = tile * kTileRows, R = min(kTileRows, n - r0);
    for (int k = tid; k <= kTileRows; k += blockDim.x) rp[buf][k] = __ldg(S.row_ptr + r0 + min(k, R));
  };
  auto issue = [&](int buf) {
    unsigned char* base = smraw + buf * Lo.stride;
    const int s0 = rp[buf][0], s1 = rp[buf][kTileRows];
    offv[buf] = stage_range(base, S.val, 9ll * s0, 9ll * s1, 8, pol_first);
    offc[buf] = stage_range(base + Lo.o_sc, S.col, s0, s1, 4, pol_first);
  };
  double dacc = 0.0;
  int tile = blockIdx.x;
  if (tile < ntiles) {
    load_rp(tile, 0);
    __syncthreads();
    issue(0);
  }
  cp_async_commit();
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int buf = it & 1;
    const int t1 = tile + gridDim.x;
    if (t1 < ntiles) {
      load_rp(t1, buf ^ 1);
      __syncthreads();
      issue(buf ^ 1);
    }
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    const int r0 = tile * kTileRows, R = min(kTileRows, n - r0);
    const unsigned char* base = smraw + buf * Lo.stride;
    const double* sv = reinterpret_cast<const double*>(base) + offv[buf];
    const int* scl = reinterpret_cast<const int*>(base + Lo.o_sc) + offc[buf];
    const int s0 = rp[buf][0], nS = rp[buf][kTileRows] - s0;
    const int ni = 3 * nS;
#pragma unroll 4
    for (int k = tid; k < ni; k += blockDim.x) {
      const int b = k / 3, r = k - 3 * (k / 3);
      const double* a = sv + 9 * b + 3 * r;
      const double* __restrict__ vc = v + 3 * (size_t)scl[b];
      contrib[b][r] = fma(a[2], __ldg(vc + 2), fma(a[1], __ldg(vc + 1), a[0] * __ldg(vc)));
    }
    __syncthreads();
    if (tid < 3 * R) {
      const int row = tid / 3, r = tid - 3 * (tid / 3);
      double acc = 0.0;
      for (int b = rp[buf][row] - s0; b < rp[buf][row + 1] - s0; ++b) acc += contrib[b][r];
      if (crp) {
        for (int s2 = __ldg(crp + r0 + row); s2 < __ldg(crp + r0 + row + 1); ++s2) {
          const double* a = C.val + 9 * (size_t)s2 + 3 * r;
          const double* vc = v + 3 * (size_t)__ldg(C.col + s2);
          acc += fma(a[2], vc[2], fma(a[1], vc[1], a[0] * vc[0]));
        }
      }
      y[3 * (size_t)(r0 + row) + r] = acc;
      if (DOT) dacc += v[3 * (size_t)(r0 + row) + r] * acc;
    }
    __syncthreads();
  }
  if (DOT) {
    __shared__ double sh[kSpmvThreads / 32];
    __shared__ bool last;
    const double bs = block_sum<kSpmvThreads>(dacc, sh);
    if (threadIdx.x == 0) {
      partials[blockIdx.x] = bs;
      __threadfence();
      last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
      __threadfence();
      double t = 0.0;
      for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t += partials[i];
      t = block_sum<kSpmvThreads>(t, sh);
      if (threadIdx.x == 0) {
        sc->pq = t;
        sc->alpha = sc->rz / t;
        *counter = 0u;
      }
    }
  }
}

template <bool DOT>
static int spmv_sf_grid(const Bsr& S, size_t& smem) {
  SfLayout Lo;
  Lo.init(S.tile_cap_s);
  smem = Lo.total;
  static int per_sm[2] = {-1, -1};
  static size_t smem_at[2] = {0, 0};
  const int key = DOT ? 1 : 0;
  if (per_sm[key] < 0 || smem_at[key] != smem) {
    if (smem > 48 * 1024)
      CK(cudaFuncSetAttribute(k_spmv_sf<DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[key], k_spmv_sf<DOT>, kSpmvThreads, smem));
    smem_at[key] = smem;
  }
  if (per_sm[key] <= 0) return 0;
  return std::max(1, std::min(per_sm[key] * num_sms(), ceil_div((long long)S.n, kTileRows)));
}

static bool spmv_sf_usable(const Bsr& S) {
  return !S.m_row_ptr && S.tile_cap_s > 0 && S.tile_cap_s <= 2048 && S.r0 == 0 && S.row_end() == S.n;
}

void spmv_prepare(const Bsr& S) {  // occupancy / smem attribute outside any stream capture
  if (!spmv_sf_usable(S)) return;
  size_t sm = 0;
  (void)spmv_sf_grid<false>(S, sm);
  (void)spmv_sf_grid<true>(S, sm);
}

void spmv_init_grids() {  // occupancy queries outside any stream capture (called by bal_init)
  Bsr one;
  one.n = 1;
  (void)spmv_grid<false, false>(one);
  (void)spmv_grid<true, false>(one);
  (void)spmv_grid<false, true>(one);
}

void launch_spmv(cudaStream_t st, const Bsr& S, const Bsr& C, const double* v, double* y) {
  if (S.n <= 0) return;
  if (ts_usable(S)) {
    launch_spmv_ts(st, S, C, v, y, S.ts->part, true);
    return;
  }
  if (spmv_sf_usable(S)) {
    size_t sm = 0;
    const int g = spmv_sf_grid<false>(S, sm);
    if (g > 0) {
      k_spmv_sf<false><<<g, kSpmvThreads, sm, st>>>(S, C, v, y, nullptr, nullptr, nullptr);
      CK(cudaGetLastError());
      return;
    }
  }
  const int blocks = spmv_grid<false, false>(S);
  k_spmv<false, false><<<blocks, kSpmvThreads, 0, st>>>(S, C, nullptr, v, y, nullptr, nullptr, nullptr, nullptr);
  CK(cudaGetLastError());
}

void launch_spmv_dot(cudaStream_t st, const Bsr& S, const Bsr& C, const double* v, double* y, double* partials,
                     unsigned* counter, PcgScal* sc) {
  if (spmv_sf_usable(S)) {
    size_t sm = 0;
    const int g = spmv_sf_grid<true>(S, sm);
    if (g > 0) {
      k_spmv_sf<true><<<g, kSpmvThreads, sm, st>>>(S, C, v, y, partials, counter, sc);
      CK(cudaGetLastError());
      return;
    }
  }
  const int blocks = spmv_grid<true, false>(S);
  k_spmv<true, false><<<blocks, kSpmvThreads, 0, st>>>(S, C, nullptr, v, y, partials, counter, sc, nullptr);
  CK(cudaGetLastError());
}

void launch_spmv_masked(cudaStream_t st, const Bsr& S, const Bsr& C, const int* grp, const double* v, double* y,
                        const GrpScal* gs) {
  const int blocks = spmv_grid<false, true>(S);
  k_spmv<false, true><<<blocks, kSpmvThreads, 0, st>>>(S, C, grp, v, y, nullptr, nullptr, nullptr, gs);
  CK(cudaGetLastError());
}

__global__ void __launch_bounds__(kVecThreads)
k_pcg_init(int n, const double* __restrict__ b, const double* __restrict__ Ax0, const double* __restrict__ dinv,
           double* __restrict__ r, double* __restrict__ z, double* __restrict__ p, double* partials,
           unsigned* counter, PcgScal* sc, double* hist) {
  double loc[3] = {0.0, 0.0, 0.0};  // rz, rr, bb
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double rr[3], bb[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      bb[c] = b[3 * (size_t)i + c];
      rr[c] = bb[c] - Ax0[3 * (size_t)i + c];
      r[3 * (size_t)i + c] = rr[c];
    }
    double z0, z1, z2;
    dinv_apply(dinv, i, rr[0], rr[1], rr[2], z0, z1, z2);
    z[3 * (size_t)i] = z0; z[3 * (size_t)i + 1] = z1; z[3 * (size_t)i + 2] = z2;
    p[3 * (size_t)i] = z0; p[3 * (size_t)i + 1] = z1; p[3 * (size_t)i + 2] = z2;
    loc[0] += rr[0] * z0 + rr[1] * z1 + rr[2] * z2;
    loc[1] += rr[0] * rr[0] + rr[1] * rr[1] + rr[2] * rr[2];
    loc[2] += bb[0] * bb[0] + bb[1] * bb[1] + bb[2] * bb[2];
  }
  double tot[3];
  if (last_block_reduce<3, kVecThreads>(loc, partials, counter, tot) && threadIdx.x == 0) {
    sc->rz = tot[0];
    sc->rr = tot[1];
    sc->bnorm = sqrt(tot[2]);
    sc->k = 0;
    sc->stop = -1;
    sc->done = 0;
    sc->dec = 0.0;
    hist[0] = sqrt(tot[1]);
    hist[sc->hcap] = 0.0;
    pcg_stop_check(sc, hist);
  }
}

void launch_pcg_init(cudaStream_t st, int n, const double* b, const double* Ax0, const double* dinv, double* r,
                     double* z, double* p, double* partials, unsigned* counter, PcgScal* sc, double* hist) {
  k_pcg_init<<<kVecBlocks, kVecThreads, 0, st>>>(n, b, Ax0, dinv, r, z, p, partials, counter, sc, hist);
  CK(cudaGetLastError());
}

__global__ void __launch_bounds__(kVecThreads)
k_pcg_update(int n, const double* __restrict__ dinv, const double* __restrict__ p, const double* __restrict__ q,
             double* __restrict__ x, double* __restrict__ r, double* __restrict__ z, double* partials,
             unsigned* counter, PcgScal* sc, double* hist) {
  if (sc->done) return;
  const double alpha = sc->alpha;
  double loc[2] = {0.0, 0.0};  // rz, rr
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
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
    loc[0] += rr[0] * z0 + rr[1] * z1 + rr[2] * z2;
    loc[1] += rr[0] * rr[0] + rr[1] * rr[1] + rr[2] * rr[2];
  }
  double tot[2];
  if (last_block_reduce<2, kVecThreads>(loc, partials, counter, tot) && threadIdx.x == 0) {
    sc->dec += 0.5 * alpha * sc->rz;  // phi(x + alpha p) = phi(x) - alpha rho / 2
    sc->beta = (sc->rz != 0.0) ? tot[0] / sc->rz : 0.0;
    sc->rz = tot[0];
    sc->rr = tot[1];
    const int k = sc->k + 1;
    sc->k = k;
    hist[k] = sqrt(tot[1]);
    hist[sc->hcap + k] = sc->dec;
    pcg_stop_check(sc, hist);
  }
}

void launch_pcg_update(cudaStream_t st, int n, const double* dinv, const double* p, const double* q, double* x,
                       double* r, double* z, double* partials, unsigned* counter, PcgScal* sc, double* hist) {
  k_pcg_update<<<kVecBlocks, kVecThreads, 0, st>>>(n, dinv, p, q, x, r, z, partials, counter, sc, hist);
  CK(cudaGetLastError());
}

__global__ void k_pcg_pupdate(int n3, const double* __restrict__ z, double* __restrict__ p, const PcgScal* sc) {
  if (sc->done) return;
  const double beta = sc->beta;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n3; j += gridDim.x * blockDim.x) p[j] = z[j] + beta * p[j];
}

// Fused update + p-update (one kernel per PCG iteration after the SpMV): x += alpha p, r -= alpha q,
// z = D^{-1} r kept in registers (never written), block partials of r.z and r.r, a grid-wide
// barrier (cooperative launch: the grid is co-resident), every CTA re-reduces the partials in the
// same fixed order (identical beta everywhere, deterministic), CTA 0 updates the scalars and the
// App. B stop test, then p = z + beta p.  Saves the z round trip and one launch per iteration.
template <int kFuseMax>  // nodes per thread held in registers
__global__ void __launch_bounds__(kVecThreads)
k_pcg_update_fused(int n, const double* __restrict__ dinv, double* __restrict__ p, const double* __restrict__ q,
                   double* __restrict__ x, double* __restrict__ r, double* partials, PcgScal* sc, double* hist) {
  if (sc->done) return;  // read by every CTA before CTA 0 can write it (after the barrier)
  const double alpha = sc->alpha, rz_old = sc->rz;
  const int T = gridDim.x * blockDim.x, t = blockIdx.x * blockDim.x + threadIdx.x;
  double z[kFuseMax][3];
  double loc0 = 0.0, loc1 = 0.0;
#pragma unroll
  for (int u = 0; u < kFuseMax; ++u) {
    const int i = t + u * T;
    z[u][0] = z[u][1] = z[u][2] = 0.0;
    if (i < n) {
      double rr[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const size_t j = 3 * (size_t)i + c;
        x[j] = x[j] + alpha * p[j];
        rr[c] = r[j] - alpha * q[j];
        r[j] = rr[c];
      }
      dinv_apply(dinv, i, rr[0], rr[1], rr[2], z[u][0], z[u][1], z[u][2]);
      loc0 += rr[0] * z[u][0] + rr[1] * z[u][1] + rr[2] * z[u][2];
      loc1 += rr[0] * rr[0] + rr[1] * rr[1] + rr[2] * rr[2];
    }
  }
  __shared__ double sh[kVecThreads / 32];
  const double b0 = block_sum<kVecThreads>(loc0, sh);
  const double b1 = block_sum<kVecThreads>(loc1, sh);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = b0;
    partials[2 * blockIdx.x + 1] = b1;
  }
  cooperative_groups::this_grid().sync();
  double t0 = 0.0, t1 = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    t0 += partials[2 * b];
    t1 += partials[2 * b + 1];
  }
  const double rz = block_sum<kVecThreads>(t0, sh);
  const double rr2 = block_sum<kVecThreads>(t1, sh);
  const double beta = (rz_old != 0.0) ? rz / rz_old : 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->dec += 0.5 * alpha * rz_old;
    sc->beta = beta;
    sc->rz = rz;
    sc->rr = rr2;
    const int k = sc->k + 1;
    sc->k = k;
    hist[k] = sqrt(rr2);
    hist[sc->hcap + k] = sc->dec;
    pcg_stop_check(sc, hist);
  }
#pragma unroll
  for (int u = 0; u < kFuseMax; ++u) {
    const int i = t + u * T;
    if (i < n) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const size_t j = 3 * (size_t)i + c;
        p[j] = z[u][c] + beta * p[j];
      }
    }
  }
}

// grid and variant (nodes per thread) for the fused update: the smallest register footprint whose
// co-resident grid holds n nodes; 0 when none does (caller falls back to update + p-update)
static int fused_per_sm(int K) {
  static int per[2] = {-1, -1};
  const int i = K == 4 ? 0 : 1;
  if (per[i] < 0) {
    if (K == 4) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per[i], k_pcg_update_fused<4>, kVecThreads, 0));
    else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per[i], k_pcg_update_fused<8>, kVecThreads, 0));
  }
  return per[i];
}

int pcg_fused_grid(int n, int* kvariant) {
  static const bool off = getenv("BAL_PCG_UNFUSED") != nullptr;
  if (off) return 0;
  for (int K : {4, 8}) {
    const int per_sm = fused_per_sm(K);
    const long long cap = (long long)per_sm * num_sms() * kVecThreads * K;
    if (per_sm > 0 && n <= cap) {
      if (kvariant) *kvariant = K;
      return std::min(per_sm * num_sms(), std::max(1, ceil_div((long long)n, (long long)kVecThreads * K)));
    }
  }
  return 0;
}

void launch_pcg_update_fused(cudaStream_t st, int grid, int n, const double* dinv, double* p, const double* q,
                             double* x, double* r, double* partials, PcgScal* sc, double* hist) {
  int K = 8;
  (void)pcg_fused_grid(n, &K);
  void* args[] = {&n, &dinv, &p, &q, &x, &r, &partials, &sc, &hist};
  const void* fn = K == 4 ? (const void*)k_pcg_update_fused<4> : (const void*)k_pcg_update_fused<8>;
  CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kVecThreads), args, 0, st));
}

void launch_pcg_pupdate(cudaStream_t st, int n, const double* z, double* p, const PcgScal* sc) {
  k_pcg_pupdate<<<kVecBlocks, kVecThreads, 0, st>>>(3 * n, z, p, sc);
  CK(cudaGetLastError());
}

// ---------------------------------------------------------------------------------------------
// Chronopoulos-Gear block-Jacobi PCG (one grid-wide reduction per iteration; same iterates as the
// textbook recurrences in exact arithmetic, oracle.linalg.pcg_cg is its parity partner):
//   init:  r_0 = b - A x_0, u_0 = M^-1 r_0, p_-1 = s_-1 = 0;
//   SpMV k (k_spmv_ts DOT): w_k = A u_k, and its last CTA reduces (r_k,u_k), (r_k,r_k), (w_k,u_k),
//          runs the App. B stop test on ||r_k|| and sets beta_k, alpha_k (cg_scalars);
//   update k (this kernel): p_k = u_k + beta_k p_{k-1}, s_k = w_k + beta_k s_{k-1} (= A p_k),
//          x += alpha_k p_k, r -= alpha_k s_k, u = M^-1 r, block partials of (r,u), (r,r) for the
//          next SpMV's reduction.  w_k = the SpMV's owned rows + the cross-tile partials of row i.
__global__ void __launch_bounds__(kVecThreads)
k_cg_init(int n, const double* __restrict__ b, const double* __restrict__ Ax0, const double* __restrict__ dinv,
          double* __restrict__ r, double* __restrict__ u, double* __restrict__ p, double* __restrict__ s,
          double* __restrict__ upart, double* partials, unsigned* counter, PcgScal* sc, double* hist,
          const double* __restrict__ x) {
  double g = 0.0, rr = 0.0, bb = 0.0, xx = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double rv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const size_t j = 3 * (size_t)i + c;
      const double bj = b[j];
      rv[c] = bj - Ax0[j];
      r[j] = rv[c];
      p[j] = 0.0;
      s[j] = 0.0;
      bb += bj * bj;
      if (x) xx += x[j] * x[j];
    }
    double u0, u1, u2;
    dinv_apply(dinv, i, rv[0], rv[1], rv[2], u0, u1, u2);
    u[3 * (size_t)i] = u0;
    u[3 * (size_t)i + 1] = u1;
    u[3 * (size_t)i + 2] = u2;
    g += rv[0] * u0 + rv[1] * u1 + rv[2] * u2;
    rr += rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2];
  }
  __shared__ double sh[kVecThreads / 32];
  const double bg = block_sum<kVecThreads>(g, sh);
  const double br = block_sum<kVecThreads>(rr, sh);
  const double bx = x ? block_sum<kVecThreads>(xx, sh) : 0.0;
  if (threadIdx.x == 0) {
    upart[2 * blockIdx.x] = bg;
    upart[2 * blockIdx.x + 1] = br;
    if (x) upart[2 * kVecBlocks + blockIdx.x] = bx;
  }
  const double loc[1] = {bb};
  double tot[1];
  if (last_block_reduce<1, kVecThreads>(loc, partials, counter, tot) && threadIdx.x == 0) {
    sc->bnorm = sqrt(tot[0]);
    if (sc->crit == 1) sc->tol = fmin(0.5, sqrt(sc->bnorm));  // App. B (i): min(0.5, sqrt||grad E||) ||grad E||
    sc->k = 0;
    sc->stop = -1;
    sc->done = 0;
    sc->dec = 0.0;
    sc->rz = sc->alpha = sc->beta = 0.0;
  }
}

void launch_cg_init(cudaStream_t st, int n, const double* b, const double* Ax0, const double* dinv, double* r,
                    double* u, double* p, double* s, double* upart, double* partials, unsigned* counter,
                    PcgScal* sc, double* hist, const double* x) {
  k_cg_init<<<kVecBlocks, kVecThreads, 0, st>>>(n, b, Ax0, dinv, r, u, p, s, upart, partials, counter, sc, hist, x);
  CK(cudaGetLastError());
}

// Two nodes per thread: their 6 consecutive doubles of every vector and 12 of D^-1 are read and
// written as 16-byte vectors (node pairs start 48 B apart, so every access is 16-byte aligned).
template <int NP>
BAL_D void cg_update_nodes(int i0, const double* __restrict__ dinv, const int* __restrict__ pin_ptr,
                           const double* __restrict__ part, const double* __restrict__ w, double* __restrict__ u,
                           double* __restrict__ p, double* __restrict__ s, double* __restrict__ x,
                           double* __restrict__ r, double alpha, double beta, double& g, double& rr, double& xx) {
  constexpr int ND = 3 * NP;
  const size_t d0 = 3 * (size_t)i0;
  double wv[ND], uv[ND], pv[ND], sv[ND], xv[ND], rv[ND];
  if (NP == 2) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double2 a = reinterpret_cast<const double2*>(w + d0)[k];
      const double2 b = reinterpret_cast<const double2*>(u + d0)[k];
      const double2 c = reinterpret_cast<const double2*>(p + d0)[k];
      const double2 d = reinterpret_cast<const double2*>(s + d0)[k];
      const double2 e = reinterpret_cast<const double2*>(x + d0)[k];
      const double2 f = reinterpret_cast<const double2*>(r + d0)[k];
      wv[2 * k] = a.x; wv[2 * k + 1] = a.y;
      uv[2 * k] = b.x; uv[2 * k + 1] = b.y;
      pv[2 * k] = c.x; pv[2 * k + 1] = c.y;
      sv[2 * k] = d.x; sv[2 * k + 1] = d.y;
      xv[2 * k] = e.x; xv[2 * k + 1] = e.y;
      rv[2 * k] = f.x; rv[2 * k + 1] = f.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      wv[k] = w[d0 + k]; uv[k] = u[d0 + k]; pv[k] = p[d0 + k];
      sv[k] = s[d0 + k]; xv[k] = x[d0 + k]; rv[k] = r[d0 + k];
    }
  }
  if (pin_ptr) {
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      const int e0 = pin_ptr[i0 + n], e1 = pin_ptr[i0 + n + 1];
      for (int e = e0; e < e1; ++e) {
#pragma unroll
        for (int c = 0; c < 3; ++c) wv[3 * n + c] += part[3 * (size_t)e + c];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    pv[k] = uv[k] + beta * pv[k];
    sv[k] = wv[k] + beta * sv[k];
    xv[k] = xv[k] + alpha * pv[k];
    rv[k] = rv[k] - alpha * sv[k];
    xx += xv[k] * xv[k];
  }
#pragma unroll
  for (int n = 0; n < NP; ++n) {
    dinv_apply(dinv, i0 + n, rv[3 * n], rv[3 * n + 1], rv[3 * n + 2], uv[3 * n], uv[3 * n + 1], uv[3 * n + 2]);
    g += rv[3 * n] * uv[3 * n] + rv[3 * n + 1] * uv[3 * n + 1] + rv[3 * n + 2] * uv[3 * n + 2];
    rr += rv[3 * n] * rv[3 * n] + rv[3 * n + 1] * rv[3 * n + 1] + rv[3 * n + 2] * rv[3 * n + 2];
  }
  if (NP == 2) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      reinterpret_cast<double2*>(p + d0)[k] = make_double2(pv[2 * k], pv[2 * k + 1]);
      reinterpret_cast<double2*>(s + d0)[k] = make_double2(sv[2 * k], sv[2 * k + 1]);
      reinterpret_cast<double2*>(x + d0)[k] = make_double2(xv[2 * k], xv[2 * k + 1]);
      reinterpret_cast<double2*>(r + d0)[k] = make_double2(rv[2 * k], rv[2 * k + 1]);
      reinterpret_cast<double2*>(u + d0)[k] = make_double2(uv[2 * k], uv[2 * k + 1]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      p[d0 + k] = pv[k]; s[d0 + k] = sv[k]; x[d0 + k] = xv[k]; r[d0 + k] = rv[k]; u[d0 + k] = uv[k];
    }
  }
}

__global__ void __launch_bounds__(kVecThreads)
k_cg_update(int n, const double* __restrict__ dinv, const int* __restrict__ pin_ptr, const double* __restrict__ part,
            const double* __restrict__ w, double* __restrict__ u, double* __restrict__ p, double* __restrict__ s,
            double* __restrict__ x, double* __restrict__ r, double* __restrict__ upart, PcgScal* sc) {
  if (sc->done) return;
  const double alpha = sc->alpha, beta = sc->beta;
  double g = 0.0, rr = 0.0, xx = 0.0;
  // 16-byte alignment of every vector (cudaMalloc / torch allocations); else one node per thread
  const bool vec = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(p) |
                     reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(r)) &
                    15) == 0;
  const int T = gridDim.x * blockDim.x, t = blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    const int npairs = n / 2;
    for (int q = t; q < npairs; q += T) cg_update_nodes<2>(2 * q, dinv, pin_ptr, part, w, u, p, s, x, r, alpha, beta, g, rr, xx);
    if ((n & 1) && t == T - 1) cg_update_nodes<1>(n - 1, dinv, pin_ptr, part, w, u, p, s, x, r, alpha, beta, g, rr, xx);
  } else {
    for (int i = t; i < n; i += T) cg_update_nodes<1>(i, dinv, pin_ptr, part, w, u, p, s, x, r, alpha, beta, g, rr, xx);
  }
  __shared__ double sh[kVecThreads / 32];
  const double bg = block_sum<kVecThreads>(g, sh);
  const double br = block_sum<kVecThreads>(rr, sh);
  const bool wx = sc->crit == 2;
  const double bx = wx ? block_sum<kVecThreads>(xx, sh) : 0.0;
  if (threadIdx.x == 0) {
    upart[2 * blockIdx.x] = bg;
    upart[2 * blockIdx.x + 1] = br;
    if (wx) upart[2 * kVecBlocks + blockIdx.x] = bx;
    if (blockIdx.x == 0) sc->k = sc->k + 1;  // read by the next SpMV's last CTA only
  }
}

void launch_cg_update(cudaStream_t st, int n, const double* dinv, const int* pin_ptr, const double* part,
                      const double* w, double* u, double* p, double* s, double* x, double* r, double* upart,
                      PcgScal* sc) {
  k_cg_update<<<kVecBlocks, kVecThreads, 0, st>>>(n, dinv, pin_ptr, part, w, u, p, s, x, r, upart, sc);
  CK(cudaGetLastError());
}

__global__ void __launch_bounds__(kVecThreads)
k_ws_init(int n, const int* __restrict__ grp, const double* __restrict__ b, const double* __restrict__ dinv,
          double* __restrict__ x, double* __restrict__ r, double* __restrict__ z, double* __restrict__ p,
          double* partials, unsigned* counter, GrpScal* gs) {
  __shared__ double bucket[(kVecThreads / 32) * kMaxGroups * 2];
  ws_zero_bucket(bucket, 2);
  const int G = gs->ngroups;
  const int stride = gridDim.x * blockDim.x;
  for (int base = blockIdx.x * blockDim.x; base < n; base += stride) {
    const int i = base + threadIdx.x;
    int g = -1;
    double v[2] = {0.0, 0.0};  // rz, rr
    if (i < n) {
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
  if (grp_finish<2>(bucket, partials, counter, G, tot)) {
    if (threadIdx.x < G) {
      const int g = threadIdx.x;
      gs->rz[g] = tot[0];
      gs->rr[g] = tot[1];
      gs->bnorm[g] = sqrt(tot[1]);
      gs->iters[g] = 0;
      const double rn = sqrt(tot[1]);
      gs->active[g] = (isfinite(rn) && !(rn <= gs->tol * gs->bnorm[g]) && gs->max_iters > 0) ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int any = 0;
      for (int g = 0; g < G; ++g) any |= gs->active[g];
      gs->any_active = any;
    }
  }
}

void launch_ws_init(cudaStream_t st, int n, const int* grp, const double* b, const double* dinv, double* x,
                    double* r, double* z, double* p, double* partials, unsigned* counter, GrpScal* gs) {
  k_ws_init<<<kVecBlocks, kVecThreads, 0, st>>>(n, grp, b, dinv, x, r, z, p, partials, counter, gs);
  CK(cudaGetLastError());
}

__global__ void __launch_bounds__(kVecThreads)
k_ws_dot(int n, const int* __restrict__ grp, const double* __restrict__ p, const double* __restrict__ q,
         double* partials, unsigned* counter, GrpScal* gs) {
  if (!gs->any_active) return;
  __shared__ double bucket[(kVecThreads / 32) * kMaxGroups * 1];
  ws_zero_bucket(bucket, 1);
  const int G = gs->ngroups;
  const int stride = gridDim.x * blockDim.x;
  for (int base = blockIdx.x * blockDim.x; base < n; base += stride) {
    const int i = base + threadIdx.x;
    int g = -1;
    double v[1] = {0.0};
    if (i < n) {
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
  if (grp_finish<1>(bucket, partials, counter, G, tot)) {
    if (threadIdx.x < G && gs->active[threadIdx.x]) {
      gs->pq[threadIdx.x] = tot[0];
      gs->alpha[threadIdx.x] = gs->rz[threadIdx.x] / tot[0];
    }
  }
}

void launch_ws_dot(cudaStream_t st, int n, const int* grp, const double* p, const double* q, double* partials,
                   unsigned* counter, GrpScal* gs) {
  k_ws_dot<<<kVecBlocks, kVecThreads, 0, st>>>(n, grp, p, q, partials, counter, gs);
  CK(cudaGetLastError());
}

__global__ void __launch_bounds__(kVecThreads)
k_ws_update(int n, const int* __restrict__ grp, const double* __restrict__ dinv, const double* __restrict__ p,
            const double* __restrict__ q, double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
            double* partials, unsigned* counter, GrpScal* gs) {
  if (!gs->any_active) return;
  __shared__ double bucket[(kVecThreads / 32) * kMaxGroups * 2];
  ws_zero_bucket(bucket, 2);
  const int G = gs->ngroups;
  const int stride = gridDim.x * blockDim.x;
  for (int base = blockIdx.x * blockDim.x; base < n; base += stride) {
    const int i = base + threadIdx.x;
    int g = -1;
    double v[2] = {0.0, 0.0};
    if (i < n) {
      g = grp[i];
      if (g >= 0 && gs->active[g]) {
        const double alpha = gs->alpha[g];
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
  if (grp_finish<2>(bucket, partials, counter, G, tot)) {
    if (threadIdx.x < G && gs->active[threadIdx.x]) {
      const int g = threadIdx.x;
      gs->beta[g] = tot[0] / gs->rz[g];
      gs->rz[g] = tot[0];
      gs->rr[g] = tot[1];
      gs->iters[g] += 1;
      const double rn = sqrt(tot[1]);
      const bool stop = !isfinite(rn) || rn <= gs->tol * gs->bnorm[g] || gs->iters[g] >= gs->max_iters;
      if (stop) gs->active[g] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int any = 0;
      for (int g = 0; g < G; ++g) any |= gs->active[g];
      gs->any_active = any;
    }
  }
}

void launch_ws_update(cudaStream_t st, int n, const int* grp, const double* dinv, const double* p, const double* q,
                      double* x, double* r, double* z, double* partials, unsigned* counter, GrpScal* gs) {
  k_ws_update<<<kVecBlocks, kVecThreads, 0, st>>>(n, grp, dinv, p, q, x, r, z, partials, counter, gs);
  CK(cudaGetLastError());
}

__global__ void k_ws_pupdate(int n, const int* __restrict__ grp, const double* __restrict__ z, double* __restrict__ p,
                             const GrpScal* gs) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int g = grp[i];
    if (g >= 0 && gs->active[g]) {
      const double beta = gs->beta[g];
#pragma unroll
      for (int c = 0; c < 3; ++c) p[3 * (size_t)i + c] = z[3 * (size_t)i + c] + beta * p[3 * (size_t)i + c];
    }
  }
}

void launch_ws_pupdate(cudaStream_t st, int n, const int* grp, const double* z, double* p, const GrpScal* gs) {
  k_ws_pupdate<<<kVecBlocks, kVecThreads, 0, st>>>(n, grp, z, p, gs);
  CK(cudaGetLastError());
}

// ------------------------------------------------------------------- generic reductions
__global__ void k_dot_part(int n, const double* __restrict__ a, const double* __restrict__ b, double* partials) {
  __shared__ double sh[kRedThreads / 32];
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    s += a[i] * (b ? b[i] : 1.0);
  s = block_sum<kRedThreads>(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}
__global__ void k_min_part(int n, const double* __restrict__ a, double* partials) {
  __shared__ double sh[kRedThreads / 32];
  double s = INFINITY;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s = fmin(s, a[i]);
  s = block_min<kRedThreads>(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}
__global__ void k_finish(int np, const double* partials, double* out, int is_min) {
  __shared__ double sh[kRedThreads / 32];
  double s = is_min ? INFINITY : 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s = is_min ? fmin(s, partials[i]) : s + partials[i];
  s = is_min ? block_min<kRedThreads>(s, sh) : block_sum<kRedThreads>(s, sh);
  if (threadIdx.x == 0) *out = s;
}

void launch_dot(cudaStream_t st, int n, const double* a, const double* b, double* partials, double* out) {
  k_dot_part<<<kRedBlocks, kRedThreads, 0, st>>>(n, a, b, partials);
  k_finish<<<1, kRedThreads, 0, st>>>(kRedBlocks, partials, out, 0);
  CK(cudaGetLastError());
}
void launch_sum(cudaStream_t st, int n, const double* a, double* partials, double* out) {
  launch_dot(st, n, a, nullptr, partials, out);
}
void launch_min(cudaStream_t st, int n, const double* a, double* partials, double* out) {
  k_min_part<<<kRedBlocks, kRedThreads, 0, st>>>(n, a, partials);
  k_finish<<<1, kRedThreads, 0, st>>>(kRedBlocks, partials, out, 1);
  CK(cudaGetLastError());
}

__global__ void k_axpy(int n, double alpha, const double* __restrict__ x, const double* __restrict__ y,
                       double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = y[i] + alpha * x[i];
}
void launch_axpy(cudaStream_t st, int n, double alpha, const double* x, const double* y, double* out) {
  k_axpy<<<kVecBlocks, kVecThreads, 0, st>>>(n, alpha, x, y, out);
  CK(cudaGetLastError());
}

__global__ void k_apply_dinv(int nn, const double* __restrict__ dinv, const double* __restrict__ r,
                             double* __restrict__ z, double scale) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += gridDim.x * blockDim.x) {
    double z0, z1, z2;
    dinv_apply(dinv, i, r[3 * (size_t)i], r[3 * (size_t)i + 1], r[3 * (size_t)i + 2], z0, z1, z2);
    z[3 * (size_t)i] = scale * z0;
    z[3 * (size_t)i + 1] = scale * z1;
    z[3 * (size_t)i + 2] = scale * z2;
  }
}
void launch_apply_dinv(cudaStream_t st, int nn, const double* dinv, const double* r, double* z, double scale) {
  k_apply_dinv<<<kVecBlocks, kVecThreads, 0, st>>>(nn, dinv, r, z, scale);
  CK(cudaGetLastError());
}

}  // namespace bal
