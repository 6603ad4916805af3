// k_spmv.cu -- symmetric BSR3 SpMV with TMA-staged tiles (§5.1).
//
// y = (D + L + L^T + sum C_i + C_i^T) v with the static part stored symmetrically (the paper's
// D + L: lower + diagonal blocks of every row, in row order) and the per-iteration contact part
// stored as full rows.  A CTA owns a tile of kSymR consecutive block rows at a time (persistent
// grid, tiles visited in increasing order wave by wave):
//   * the tile's stored blocks (one contiguous range of lval / l_col) are streamed into shared
//     memory by one cp.async.bulk (TMA, 1-D) per array, completing on an mbarrier, NST-stage ring,
//     L2 evict_first -- no per-thread global loads for the dominant byte stream;
//   * each stored block A_ij is used twice from shared memory: A_ij v_j for row i, and, when row j
//     lies in the same tile (the in-tile mirror, ~57 % of the blocks at 64 rows on C4), A_ij^T v_i
//     for row j -- so that block leaves HBM once and is never re-read;
//   * the remaining mirror blocks (row j in this tile, i in a later tile) are gathered from global
//     memory with L2 evict_last: their own tile streams them later, from L2;
//   * every row sums its contributions in a fixed order (stored ascending column, mirror ascending
//     row, contact ascending column) -- bitwise deterministic, atomic-free, and bitwise identical
//     to the per-item arithmetic of the generic kernel (k_linalg.cu).
// Fused epilogue (DOT): p^T A p partials, last-CTA ticket reduce, alpha = rz / pAp on the device.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace bal {

namespace {

BAL_D unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

BAL_D void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
BAL_D void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
BAL_D void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
BAL_D void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
BAL_D unsigned long long pol_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
BAL_D unsigned long long pol_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
BAL_D double ldg_hint(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// dynamic shared memory layout (bytes), shared by host (size) and device (offsets)
struct SymLayout {
  int cap, ocap;
  size_t o_val, val_stride, o_col, col_stride, o_cs, o_ct, o_co, o_sv, o_rp, o_lrow, o_smi, total;
  BAL_HD SymLayout(int cap_, int ocap_, int nst) : cap(cap_), ocap(ocap_) {
    auto up = [](size_t x) { return (x + 127) & ~(size_t)127; };
    o_val = 128;  // [0, 128): mbarriers
    val_stride = up((size_t)cap * 72 + 16);
    o_col = o_val + nst * val_stride;
    col_stride = up((size_t)cap * 4 + 16);
    o_cs = o_col + nst * col_stride;
    o_ct = o_cs + up((size_t)cap * 24);
    o_co = o_ct + up((size_t)cap * 24);
    o_sv = o_co + up((size_t)(ocap > 1 ? ocap : 1) * 24);
    o_rp = o_sv + up((size_t)kSymR * 24);
    o_lrow = o_rp + up(3 * (size_t)(kSymR + 1) * 4);
    o_smi = o_lrow + up((size_t)cap * 2);
    total = o_smi + up((size_t)cap * 2);
  }
};

}  // namespace

template <bool DOT, int NST>
__global__ void __launch_bounds__(kSymThreads)
k_spmv_sym(Bsr S, Bsr C, const double* __restrict__ v, double* __restrict__ y, double* partials, unsigned* counter,
           PcgScal* sc) {
  if (DOT && sc->done) return;
  extern __shared__ __align__(128) unsigned char sm[];
  const SymLayout Lo(S.tcap, S.tocap, NST);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  double* cs = reinterpret_cast<double*>(sm + Lo.o_cs);
  double* ct = reinterpret_cast<double*>(sm + Lo.o_ct);
  double* co = reinterpret_cast<double*>(sm + Lo.o_co);
  double* sv = reinterpret_cast<double*>(sm + Lo.o_sv);
  int* rp = reinterpret_cast<int*>(sm + Lo.o_rp);  // [3][kSymR + 1]: stored, in-tile mirror, out mirror
  unsigned short* lrow = reinterpret_cast<unsigned short*>(sm + Lo.o_lrow);
  unsigned short* smi = reinterpret_cast<unsigned short*>(sm + Lo.o_smi);
  const int n = S.n;
  const int tid = threadIdx.x;
  const int t0 = S.r0 / kSymR, ntiles = (S.row_end() + kSymR - 1) / kSymR;
  const int G = gridDim.x;
  const unsigned long long pf = pol_evict_first(), pl = pol_evict_last();
  const int* crp = C.nnzb > 0 ? C.row_ptr : nullptr;

  // producer: one thread streams tile t's stored blocks + columns into stage b
  auto issue = [&](int t, int b) {
    const int r0 = t * kSymR, r1 = min(S.row_end(), r0 + kSymR);
    const int s0 = __ldg(S.row_ptr + r0), s1 = __ldg(S.row_ptr + r1);
    const size_t a0 = (72ull * s0) & ~15ull, e0 = (72ull * s1 + 15) & ~15ull;
    const size_t c0 = (4ull * s0) & ~15ull, f0 = (4ull * s1 + 15) & ~15ull;
    const unsigned bv = (unsigned)(e0 - a0), bc = (unsigned)(f0 - c0);
    mbar_expect_tx(bar + b, bv + bc);
    bulk_g2s(sm + Lo.o_val + b * Lo.val_stride, reinterpret_cast<const unsigned char*>(S.val) + a0, bv, bar + b, pf);
    bulk_g2s(sm + Lo.o_col + b * Lo.col_stride, reinterpret_cast<const unsigned char*>(S.col) + c0, bc, bar + b, pf);
  };

  if (tid == 0) {
    for (int b = 0; b < NST; ++b) mbar_init(bar + b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int b = 0; b < NST; ++b)
      if (t0 + blockIdx.x + b * G < ntiles) issue(t0 + blockIdx.x + b * G, b);

  double dacc = 0.0;
  int it = 0;
  for (int tile = t0 + blockIdx.x; tile < ntiles; tile += G, ++it) {
    const int b = it % NST;
    const unsigned parity = (unsigned)((it / NST) & 1);
    const int r0 = tile * kSymR;
    const int R = min(kSymR, S.row_end() - r0);
    // ---- phase 0 (while the bulk copy is in flight): row pointers, the tile's v rows
    for (int t = tid; t < 3 * (kSymR + 1); t += kSymThreads) {
      const int L = t / (kSymR + 1), k = t - L * (kSymR + 1);
      const int* p = L == 0 ? S.row_ptr : (L == 1 ? S.mi_row_ptr : S.mo_row_ptr);
      rp[t] = k <= R ? __ldg(p + r0 + k) : 0;
    }
    for (int t = tid; t < 3 * R; t += kSymThreads) sv[t] = __ldg(v + 3 * (size_t)r0 + t);
    __syncthreads();
    const int s0 = rp[0], nb = rp[R] - s0;
    const int* rpi = rp + (kSymR + 1);
    const int* rpo = rp + 2 * (kSymR + 1);
    const int m0 = rpi[0], nmi = rpi[R] - m0;
    const int o0 = rpo[0], no = rpo[R] - o0;
    for (int r = tid; r < R; r += kSymThreads)
      for (int q = rp[r] - s0; q < rp[r + 1] - s0; ++q) lrow[q] = (unsigned short)r;
    for (int t = tid; t < nmi; t += kSymThreads) smi[t] = __ldg(S.mi_loc + m0 + t);
    // ---- phase C: out-of-tile mirror blocks A_ij (i in a later tile): gathered, L2 evict_last
    for (int m = tid; m < no; m += kSymThreads) {
      const int pos = __ldg(S.mo_pos + o0 + m), i = __ldg(S.mo_col + o0 + m);
      const double* a = S.val + 9 * (size_t)pos;
      double A[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) A[k] = ldg_hint(a + k, pl);
      const double* vi = v + 3 * (size_t)i;
      const double x0 = __ldg(vi), x1 = __ldg(vi + 1), x2 = __ldg(vi + 2);
#pragma unroll
      for (int c = 0; c < 3; ++c) co[3 * m + c] = fma(A[6 + c], x2, fma(A[3 + c], x1, A[c] * x0));
    }
    __syncthreads();
    mbar_wait(bar + b, parity);
    const double* sval = reinterpret_cast<const double*>(sm + Lo.o_val + b * Lo.val_stride) + (s0 & 1);
    const int* scol = reinterpret_cast<const int*>(sm + Lo.o_col + b * Lo.col_stride) + (s0 & 3);
    // ---- phase A/B: every stored block from shared memory: A v_j (row i), A^T v_i (row j, in-tile)
    for (int q = tid; q < nb; q += kSymThreads) {
      const double* A = sval + 9 * q;
      const int j = scol[q];
      const int il = lrow[q];
      const int jl = j - r0;
      double x0, x1, x2;
      if (jl >= 0) {
        x0 = sv[3 * jl];
        x1 = sv[3 * jl + 1];
        x2 = sv[3 * jl + 2];
      } else {
        const double* vj = v + 3 * (size_t)j;
        x0 = __ldg(vj);
        x1 = __ldg(vj + 1);
        x2 = __ldg(vj + 2);
      }
      double a[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) a[k] = A[k];
#pragma unroll
      for (int r = 0; r < 3; ++r) cs[3 * q + r] = fma(a[3 * r + 2], x2, fma(a[3 * r + 1], x1, a[3 * r] * x0));
      if (jl >= 0 && jl != il) {
        const double w0 = sv[3 * il], w1 = sv[3 * il + 1], w2 = sv[3 * il + 2];
#pragma unroll
        for (int c = 0; c < 3; ++c) ct[3 * q + c] = fma(a[6 + c], w2, fma(a[3 + c], w1, a[c] * w0));
      }
    }
    __syncthreads();
    // ---- phase D: fixed-order row sums (stored asc. column, mirror asc. row, contact asc. column)
    for (int t = tid; t < 3 * R; t += kSymThreads) {
      const int row = t / 3, c = t - 3 * (t / 3);
      double acc = 0.0;
      for (int q = rp[row] - s0; q < rp[row + 1] - s0; ++q) acc += cs[3 * q + c];
      for (int e = rpi[row] - m0; e < rpi[row + 1] - m0; ++e) acc += ct[3 * smi[e] + c];
      for (int m = rpo[row] - o0; m < rpo[row + 1] - o0; ++m) acc += co[3 * m + c];
      if (crp) {
        const int gr = r0 + row;
        for (int s2 = __ldg(crp + gr); s2 < __ldg(crp + gr + 1); ++s2) {
          const double* a = C.val + 9 * (size_t)s2 + 3 * c;
          const double* vc = v + 3 * (size_t)__ldg(C.col + s2);
          acc += fma(a[2], __ldg(vc + 2), fma(a[1], __ldg(vc + 1), a[0] * __ldg(vc)));
        }
      }
      y[3 * (size_t)r0 + t] = acc;
      if (DOT) dacc += sv[t] * acc;
    }
    __syncthreads();  // stage b, rp, sv, cs/ct/co are rewritten next
    if (tid == 0 && tile + NST * G < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile + NST * G, b);
    }
  }
  if (DOT) {
    __shared__ double sh[kSymThreads / 32];
    __shared__ bool last;
    const double bs = block_sum<kSymThreads>(dacc, sh);
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
      t = block_sum<kSymThreads>(t, sh);
      if (threadIdx.x == 0) {
        sc->pq = t;
        sc->alpha = sc->rz / t;
        *counter = 0u;
      }
    }
  }
}

namespace {
template <bool DOT>
struct SymCfg {
  int per_sm = -1;
  size_t smem = 0;
};
template <bool DOT>
SymCfg<DOT>& sym_cfg() {
  static SymCfg<DOT> c;
  return c;
}
template <bool DOT>
int sym_grid(const Bsr& S, size_t& smem) {
  const SymLayout Lo(S.tcap, S.tocap, kSymStages);
  smem = Lo.total;
  SymCfg<DOT>& c = sym_cfg<DOT>();
  if (c.per_sm < 0 || c.smem != smem) {
    auto fn = k_spmv_sym<DOT, kSymStages>;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.per_sm, fn, kSymThreads, smem));
    c.smem = smem;
  }
  if (c.per_sm <= 0) return 0;
  const int ntiles = ceil_div((long long)S.row_end(), kSymR) - S.r0 / kSymR;
  return std::max(1, std::min(c.per_sm * num_sms(), ntiles));
}
}  // namespace

bool spmv_sym_usable(const Bsr& S) {
  return S.mi_row_ptr != nullptr && S.tcap > 0 && S.r0 % kSymR == 0 && (S.r1 < 0 || S.r1 == S.n || S.r1 % kSymR == 0);
}

void spmv_sym_prepare(const Bsr& S) {  // attributes / occupancy outside any stream capture
  if (!spmv_sym_usable(S)) return;
  size_t sm = 0;
  (void)sym_grid<false>(S, sm);
  (void)sym_grid<true>(S, sm);
}

bool launch_spmv_sym(cudaStream_t st, const Bsr& S, const Bsr& C, const double* v, double* y, double* partials,
                     unsigned* counter, PcgScal* sc) {
  if (!spmv_sym_usable(S)) return false;
  size_t sm = 0;
  if (sc) {
    const int g = sym_grid<true>(S, sm);
    if (g <= 0) return false;
    k_spmv_sym<true, kSymStages><<<g, kSymThreads, sm, st>>>(S, C, v, y, partials, counter, sc);
  } else {
    const int g = sym_grid<false>(S, sm);
    if (g <= 0) return false;
    k_spmv_sym<false, kSymStages><<<g, kSymThreads, sm, st>>>(S, C, v, y, nullptr, nullptr, nullptr);
  }
  CK(cudaGetLastError());
  return true;
}

}  // namespace bal
