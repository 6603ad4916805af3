// k_spmv_ts.cu -- tile-symmetric BSR3 SpMV with cross-tile partials (§5.1).
//
// y = (D + L + L^T + sum C_i + C_i^T) v with the static part stored symmetrically (the paper's D + L:
// lower + diagonal blocks of every row, row order, 72 B values (36 B with BAL_FP32_MATRIX) + 4 B
// per block) and the
// per-iteration contact part stored as full rows.
//
// The rows are cut into tiles of consecutive rows holding at most `budget` stored blocks (<= 256
// rows).  A tile's stored blocks are one contiguous range of the value array, so a CTA streams
// them into shared memory with one 1-D TMA bulk copy (cp.async.bulk, mbarrier completion, L2
// evict_first) together with the tile's static metadata and its rows of v, kTsStages tiles ahead.
// Every stored block A_ij (i in the tile, j <= i) leaves HBM exactly once and is used from shared
// memory for both of its products:
//   * A_ij v_j  -> row i (owned by the tile);
//   * A_ij^T v_i -> row j: if j is in the tile, summed into row j's result (in-tile mirror list);
//     if j is in an earlier tile, summed per (tile, j) in a fixed order into one 3-vector
//     "partial", written to a slot of the partial buffer.  Slots are sorted by target row, so
//     the consumer of y (PCG update, or k_ts_combine for a plain product) adds
//     part[pin_ptr[j] .. pin_ptr[j+1]) to row j with coalesced reads.
// No block is read twice, nothing is gathered from global memory except v at the (deduplicated)
// out-of-tile columns (cp.async, one tile ahead) and the contact blocks; no atomics; every sum is
// in a fixed order, so the product is bitwise deterministic.
// DOT variant (single-reduction PCG, k_linalg.cu): the epilogue accumulates v^T (A v) over the
// owned rows and the partials (v_j . partial_j), and the last CTA (atomic ticket) reduces it
// together with the (r, u) and (r, r) block partials of the preceding PCG update kernel -- the
// one grid-wide reduction of a Chronopoulos-Gear PCG iteration.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "reduce.cuh"

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
      "TS_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TS_WAIT_%=;\n"
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
BAL_D void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
BAL_D void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
BAL_D void bulk_prefetch_l2(const void* src, unsigned bytes) {  // TMA prefetch into L2, no smem
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
BAL_D void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
BAL_D void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// metadata header of a tile (32 B): counts, shared-memory sizes and the tile's first row / block
struct TsHdr {
  int nb, R, ncross, ncs, ntp, r0, s0, pad;  // ncs / ntp = padded sizes of the cs / tp scratch (3-vectors)
};

// pointers into a tile's metadata (layout written by ts_build).  Phase 1 writes block q's row term
// A v_j to cs[cpos[q]] (the row's terms contiguous: row il = [rpc[il], rpc[il] + rle[il])) and, for
// an off-diagonal block, its transposed term A^T v_i to tp[tslot[q]] (grouped by target: in-tile
// row il = [mps[il], mps[il] + mle[il]), out-of-tile target x = [xps[x], xps[x] + xle[x])), every
// group in ascending block order.  Groups are placed at odd 3-vector strides (a padding slot after
// each even-length group), so one thread per row reading its group's k-th term hits distinct shared
// memory banks on regular meshes.
struct TsMeta {
  const TsHdr* h;
  const int* gx;               // [ncross] global column of each out-of-tile target (ascending)
  const int* pslot;            // [ncross] partial slot of (this tile, target)
  const unsigned* code;        // [nb] il | jref << 8 | kind << 24 (kind 0 diag, 1 in-tile, 2 cross)
  const unsigned short* cpos;  // [nb]
  const unsigned short* tslot; // [nb] (unused for diagonal blocks)
  const unsigned short *rpc, *rle, *mps, *mle;  // [R]
  const unsigned short *xps, *xle;              // [ncross]
  BAL_HD explicit TsMeta(const unsigned char* m) {
    h = reinterpret_cast<const TsHdr*>(m);
    gx = reinterpret_cast<const int*>(m + sizeof(TsHdr));
    pslot = gx + h->ncross;
    code = reinterpret_cast<const unsigned*>(pslot + h->ncross);
    cpos = reinterpret_cast<const unsigned short*>(code + h->nb);
    tslot = cpos + h->nb;
    rpc = tslot + h->nb;
    rle = rpc + h->R;
    mps = rle + h->R;
    mle = mps + h->R;
    xps = mle + h->R;
    xle = xps + h->ncross;
  }
};

inline size_t ts_meta_bytes(int nb, int R, int ncross) {
  const size_t b = sizeof(TsHdr) + 12 * (size_t)ncross + 8 * (size_t)nb + 8 * (size_t)R;
  return (b + 15) & ~(size_t)15;
}

BAL_HD size_t up128(size_t x) { return (x + 127) & ~(size_t)127; }

}  // namespace

// ------------------------------------------------------------------------------------------ plan
bool ts_build(int N, const std::vector<int>& lrow, const std::vector<int>& lcol, int budget, int val_bytes,
              TsHost& P) {
  P = TsHost();
  P.val_bytes = val_bytes;
  if (N <= 0) return false;
  // tiles: maximal runs of consecutive rows with <= budget stored blocks and <= kTsMaxRows rows
  // (one phase-1 thread per row)
  P.tile_r0.push_back(0);
  for (int r0 = 0; r0 < N;) {
    int r1 = r0 + 1;
    while (r1 < N && r1 - r0 < kTsMaxRows && lrow[r1 + 1] - lrow[r0] <= budget) ++r1;
    if (lrow[r1] - lrow[r0] >= 65536) return false;  // 16-bit local indices
    P.tile_r0.push_back(r1);
    r0 = r1;
  }
  const int ntiles = (int)P.tile_r0.size() - 1;
  P.tile_s0.resize(ntiles + 1);
  for (int t = 0; t <= ntiles; ++t) P.tile_s0[t] = lrow[P.tile_r0[t]];
  std::vector<int> xid(N, -1), cnt(N + 1, 0);
  std::vector<size_t> slot_at;  // byte offset in meta of each (tile, target) slot entry
  std::vector<int> slot_tgt;
  P.meta_off.assign(ntiles + 1, 0);
  for (int t = 0; t < ntiles; ++t) {
    const int r0 = P.tile_r0[t], r1 = P.tile_r0[t + 1], R = r1 - r0;
    const int s0 = lrow[r0], nb = lrow[r1] - s0;
    std::vector<int> gx;
    for (int s = s0; s < s0 + nb; ++s)
      if (lcol[s] < r0 && xid[lcol[s]] < 0) {
        xid[lcol[s]] = 0;
        gx.push_back(lcol[s]);
      }
    std::sort(gx.begin(), gx.end());
    const int ncross = (int)gx.size();
    if (ncross >= 65536) return false;
    for (int x = 0; x < ncross; ++x) xid[gx[x]] = x;
    std::vector<unsigned> code(nb);
    std::vector<unsigned short> cpos(nb), tslot(nb, 0xffffu), rpc(R), rle(R), mps(R), mle(R), xps(ncross),
        xle(ncross);
    std::vector<std::vector<int>> mil(R), xl(ncross);
    int ncs = 0;
    for (int il = 0; il < R; ++il) {
      const int len = lrow[r0 + il + 1] - lrow[r0 + il];
      if (len > 0xffff) return false;
      rpc[il] = (unsigned short)ncs;
      rle[il] = (unsigned short)len;
      for (int s = lrow[r0 + il]; s < lrow[r0 + il + 1]; ++s) {
        const int q = s - s0, j = lcol[s];
        cpos[q] = (unsigned short)(ncs + (s - lrow[r0 + il]));
        unsigned kind, jref;
        if (j == r0 + il) {
          kind = 0;
          jref = (unsigned)il;
        } else if (j >= r0) {
          kind = 1;
          jref = (unsigned)(j - r0);
          mil[j - r0].push_back(q);
        } else {
          kind = 2;
          jref = (unsigned)xid[j];
          xl[xid[j]].push_back(q);
        }
        code[q] = (unsigned)il | (jref << 8) | (kind << 24);
      }
      ncs += len == 0 ? 0 : (len | 1);  // odd stride between consecutive rows' groups
    }
    int pos = 0;
    for (int il = 0; il < R; ++il) {
      mps[il] = (unsigned short)pos;
      mle[il] = (unsigned short)mil[il].size();
      for (size_t k = 0; k < mil[il].size(); ++k) tslot[mil[il][k]] = (unsigned short)(pos + k);
      pos += mil[il].empty() ? 0 : ((int)mil[il].size() | 1);
    }
    for (int x = 0; x < ncross; ++x) {
      xps[x] = (unsigned short)pos;
      xle[x] = (unsigned short)xl[x].size();
      for (size_t k = 0; k < xl[x].size(); ++k) tslot[xl[x][k]] = (unsigned short)(pos + k);
      pos += xl[x].empty() ? 0 : ((int)xl[x].size() | 1);
    }
    const int ntp = pos;
    if (ncs >= 65536 || ntp >= 65536) return false;
    const size_t mb = ts_meta_bytes(nb, R, ncross);
    const size_t off = P.meta.size();
    P.meta.resize(off + mb, 0);
    unsigned char* m = P.meta.data() + off;
    TsHdr h{nb, R, ncross, ncs, ntp, r0, s0, 0};
    std::memcpy(m, &h, sizeof(h));
    size_t o = sizeof(TsHdr);
    std::memcpy(m + o, gx.data(), 4 * (size_t)ncross);
    o += 4 * (size_t)ncross;
    for (int x = 0; x < ncross; ++x) {  // partial slots filled once every tile's targets are known
      slot_at.push_back(off + o + 4 * (size_t)x);
      slot_tgt.push_back(gx[x]);
      cnt[gx[x] + 1] += 1;
    }
    o += 4 * (size_t)ncross;
    std::memcpy(m + o, code.data(), 4 * (size_t)nb);
    o += 4 * (size_t)nb;
    auto put16 = [&](const std::vector<unsigned short>& v) {
      if (!v.empty()) std::memcpy(m + o, v.data(), 2 * v.size());
      o += 2 * v.size();
    };
    for (auto* v : {&cpos, &tslot, &rpc, &rle, &mps, &mle, &xps, &xle}) put16(*v);
    P.cap_cs = std::max(P.cap_cs, ncs);
    P.cap_tp = std::max(P.cap_tp, ntp);
    P.meta_off[t + 1] = (long long)P.meta.size();
    P.cap_nb = std::max(P.cap_nb, nb);
    P.cap_rows = std::max(P.cap_rows, R);
    P.cap_x = std::max(P.cap_x, ncross);
    P.cap_meta = std::max(P.cap_meta, (int)mb);
    P.ncross_total += ncross;
    for (int x = 0; x < ncross; ++x) xid[gx[x]] = -1;
  }
  // partial slots sorted by target row, then source tile (tiles were visited in increasing order)
  P.pin_ptr.assign(N + 1, 0);
  for (int j = 0; j < N; ++j) P.pin_ptr[j + 1] = P.pin_ptr[j] + cnt[j + 1];
  std::vector<int> seen(N, 0);
  for (size_t e = 0; e < slot_at.size(); ++e) {
    const int j = slot_tgt[e];
    const int sl = P.pin_ptr[j] + seen[j]++;
    std::memcpy(P.meta.data() + slot_at[e], &sl, 4);
  }
  P.nslots = P.pin_ptr[N];
  P.ntiles = ntiles;
  // shared-memory layout of one stage: metadata | values | v rows | out-of-tile v
  P.o_meta = 0;
  P.o_val = up128((size_t)P.cap_meta);
  P.o_vt = P.o_val + up128((size_t)P.cap_nb * val_bytes + 32);
  P.o_xv = P.o_vt + up128((size_t)P.cap_rows * 24 + 32);
  P.o_crp = P.o_xv + up128((size_t)std::max(P.cap_x, 1) * 24);
  P.stage_bytes = P.o_crp + up128((size_t)(P.cap_rows + 1) * 4);
  // + the row terms (cs) and transposed terms (tp) of a tile, double-buffered across tiles
  P.o_scratch = 128 + (size_t)kTsStages * P.stage_bytes;
  P.smem = P.o_scratch + kTsScratchBufs * 24 * (size_t)(P.cap_cs + P.cap_tp + kTsContactCap);
  return true;
}

// ------------------------------------------------------------------------------------------ kernel
struct TsArgs {
  TsPlan P;
  const void* val;  // lower + diagonal blocks: double[9] (FP64) or float[9] (BAL_FP32_MATRIX)
  Bsr C;
  const double* v;
  double* y;
  double* part;
  double* dpart;
  unsigned* counter;
  PcgScal* sc;
  const double* upart;
  double* hist;
  int cpref;  // producer prefetches each tile's contact range (values, columns) into L2
};

// sum of the 3-vectors p[3b .. 3e) into (s0, s1, s2), four independent partial sums (short
// dependent chains), fixed order
BAL_D void sum3(const double* __restrict__ p, int b, int e, double& s0, double& s1, double& s2) {
  double t0 = 0.0, t1 = 0.0, t2 = 0.0, u0 = 0.0, u1 = 0.0, u2 = 0.0;
  for (; b + 2 <= e; b += 2) {
    t0 += p[3 * b];
    t1 += p[3 * b + 1];
    t2 += p[3 * b + 2];
    u0 += p[3 * b + 3];
    u1 += p[3 * b + 4];
    u2 += p[3 * b + 5];
  }
  if (b < e) {
    t0 += p[3 * b];
    t1 += p[3 * b + 1];
    t2 += p[3 * b + 2];
  }
  s0 += t0 + u0;
  s1 += t1 + u1;
  s2 += t2 + u2;
}

BAL_D void bar_consumers() {  // named barrier 1: the kTsConsumers consumer threads only
  asm volatile("bar.sync 1, %0;" ::"n"(kTsConsumers) : "memory");
}
BAL_D void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
BAL_D void cp_async_mbar_arrive(uint64_t* bar) {  // arrives when this thread's prior cp.async land
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-specialised persistent kernel: warp 0 is the producer (TMA bulk copies of metadata, values and
// v rows into a kTsStages ring; once a tile's metadata has landed, cp.async gathers of v at its
// out-of-tile columns and of its contact row pointers), warps 1.. are consumers (phase 1: one thread
// per stored block; consumer barrier; phase 2: one thread per owned row / out-of-tile target).
// Barriers per stage: full (TMA bytes), gath (32 producer lanes' cp.async), empty (consumer warps).
#ifdef BAL_TS_TIMING
__device__ unsigned long long g_ts_timing[16];
#define TS_T(k)                              \
  if (lane == 0) {                           \
    const long long t_ = clock64();          \
    tacc[k] += t_ - tlast;                   \
    tlast = t_;                              \
  }
#else
#define TS_T(k)
#endif

template <bool DOT, typename VT>
__global__ void __launch_bounds__(kTsThreads, kTsMinBlocks) k_spmv_ts(const TsArgs a) {
  const VT* aval = static_cast<const VT*>(a.val);
  if (DOT && a.sc->done) return;
#ifdef BAL_TS_TIMING
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tlast = clock64();
#endif
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* gath = full + kTsStages;
  uint64_t* empty = gath + kTsStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, first = blockIdx.x;
  const int ntl = a.P.ntiles;
  const int count = first < ntl ? (ntl - 1 - first) / G + 1 : 0;
  const int* crp = a.C.nnzb > 0 ? a.C.row_ptr : nullptr;
  auto stage = [&](int it) { return sm + 128 + (size_t)(it % kTsStages) * a.P.stage_bytes; };
  auto par = [&](int it) { return (unsigned)((it / kTsStages) & 1); };
  auto v_span = [&](int r0, int r1, uintptr_t& xa0, uintptr_t& xe1, uintptr_t& xa, uintptr_t& xe) {
    xa = reinterpret_cast<uintptr_t>(a.v + 3 * (size_t)r0);
    xe = reinterpret_cast<uintptr_t>(a.v + 3 * (size_t)r1);
    xa0 = xa & ~(uintptr_t)15;
    xe1 = xe & ~(uintptr_t)15;  // [xe1, xe) (0 or 8 bytes) is fetched by the gather
  };
  if (tid == 0) {
    for (int b = 0; b < kTsStages; ++b) {
      mbar_init(full + b, 1);
      mbar_init(gath + b, 32);
      mbar_init(empty + b, kTsConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double dacc = 0.0;
  if (warp == 0) {
    // ================================================================ producer
    const unsigned long long pf = pol_evict_first(), pl = pol_evict_last();
    constexpr int D = kTsStages - 1;  // gathers trail the bulk copies by D tiles
    int4 d0 = make_int4(0, 0, 0, 0), d1 = d0;
    int pc0 = 0, pc1 = 0;  // contact range of the tile whose bulk copies were issued last
    if (lane == 0 && count > 0) {
      d0 = __ldg(a.P.desc + first);
      d1 = __ldg(a.P.desc + first + 1);
    }
    // iteration j: gather for tile j - D (its bulk copies were issued D iterations ago), then bulk
    // copies for tile j once the consumers have released its stage
    for (int j = 0; j < count + D; ++j) {
      const int k = j - D;
      TS_T(1)
      if (lane == 0 && pc1 > pc0) {
        // the contact blocks of tile j - 1 (row-sorted contact BSR: one contiguous range) into L2, so
        // the consumers' per-block loads of them one tile later hit L2 instead of HBM
        const uintptr_t ca = reinterpret_cast<uintptr_t>(a.C.val + 9 * (size_t)pc0) & ~(uintptr_t)15;
        const uintptr_t ce = (reinterpret_cast<uintptr_t>(a.C.val + 9 * (size_t)pc1) + 15) & ~(uintptr_t)15;
        bulk_prefetch_l2(reinterpret_cast<const void*>(ca), (unsigned)(ce - ca));
        const uintptr_t ka = reinterpret_cast<uintptr_t>(a.C.col + pc0) & ~(uintptr_t)15;
        const uintptr_t ke = (reinterpret_cast<uintptr_t>(a.C.col + pc1) + 15) & ~(uintptr_t)15;
        bulk_prefetch_l2(reinterpret_cast<const void*>(ka), (unsigned)(ke - ka));
        pc0 = pc1 = 0;
      }
      if (k >= 0) {
        mbar_wait(full + k % kTsStages, par(k));
        TS_T(2)
        unsigned char* S = stage(k);
        const TsMeta M(S + a.P.o_meta);
        const int nc = M.h->ncross, R = M.h->R, r0 = M.h->r0;
        double* xv = reinterpret_cast<double*>(S + a.P.o_xv);
        for (int e = lane; e < 3 * nc; e += 32) {
          const int x = e / 3, c = e - 3 * x;
          cp_async8(xv + e, a.v + 3 * (size_t)M.gx[x] + c);
        }
        if (crp) {
          int* cr = reinterpret_cast<int*>(S + a.P.o_crp);
          for (int q = lane; q <= R; q += 32) cp_async4(cr + q, crp + r0 + q);
        }
        if (lane == 0) {
          uintptr_t xa0, xe1, xa, xe;
          v_span(r0, r0 + R, xa0, xe1, xa, xe);
          if (xe != xe1) cp_async8(S + a.P.o_vt + (xe1 - xa0), reinterpret_cast<const void*>(xe1));
        }
        cp_async_mbar_arrive(gath + k % kTsStages);
        TS_T(3)
      }
      if (j < count) {
        TS_T(7)
        if (j >= kTsStages) mbar_wait(empty + j % kTsStages, par(j - kTsStages));
        TS_T(0)
        if (lane == 0) {
          unsigned char* S = stage(j);
          uint64_t* fb = full + j % kTsStages;
          const long long m0 = 16ll * d0.x, m1 = 16ll * d1.x;
          const uintptr_t va = reinterpret_cast<uintptr_t>(aval + 9 * (size_t)d0.y);
          const uintptr_t ve = reinterpret_cast<uintptr_t>(aval + 9 * (size_t)d1.y);
          const uintptr_t va0 = va & ~(uintptr_t)15, ve1 = (ve + 15) & ~(uintptr_t)15;
          uintptr_t xa0, xe1, xa, xe;
          v_span(d0.z, d1.z, xa0, xe1, xa, xe);
          const unsigned bm = (unsigned)(m1 - m0), bv = (unsigned)(ve1 - va0), bx = (unsigned)(xe1 - xa0);
          mbar_expect_tx(fb, bm + bv + bx);
          bulk_g2s(S + a.P.o_meta, a.P.meta + m0, bm, fb, pf);
          bulk_g2s(S + a.P.o_val, reinterpret_cast<const void*>(va0), bv, fb, pf);
          if (bx) bulk_g2s(S + a.P.o_vt, reinterpret_cast<const void*>(xa0), bx, fb, pl);
          if (crp && a.cpref) {  // consumed at the next iteration (load latency off the critical path)
            pc0 = __ldg(crp + d0.z);
            pc1 = __ldg(crp + d1.z);
          }
          if (j + 1 < count) {  // next tile's descriptors, off the critical path
            const int t = first + (j + 1) * G;
            d0 = __ldg(a.P.desc + t);
            d1 = __ldg(a.P.desc + t + 1);
          }
        }
        __syncwarp();
      }
    }
  } else {
    // ================================================================ consumers
    const int ct = tid - 32;  // consumer thread index
    for (int it = 0; it < count; ++it) {
      TS_T(7)
      mbar_wait(full + it % kTsStages, par(it));
      TS_T(4)
      mbar_wait(gath + it % kTsStages, par(it));
      TS_T(5)
      const unsigned char* S = stage(it);
      const TsMeta M(S + a.P.o_meta);
      const int R = M.h->R, nc = M.h->ncross, r0 = M.h->r0, s0 = M.h->s0, nb = M.h->nb;
      const uintptr_t va = reinterpret_cast<uintptr_t>(aval + 9 * (size_t)s0);
      const VT* vals = reinterpret_cast<const VT*>(S + a.P.o_val + (va & 15));
      uintptr_t xa0, xe1, xa, xe;
      v_span(r0, r0 + R, xa0, xe1, xa, xe);
      const double* vt = reinterpret_cast<const double*>(S + a.P.o_vt + (xa - xa0));
      const double* xv = reinterpret_cast<const double*>(S + a.P.o_xv);
      // double-buffered scratch: [nb][3] A v_j (row terms) then [noff][3] A^T v_i (slot order)
      double* cs = reinterpret_cast<double*>(sm + a.P.o_scratch) +
                   (size_t)(it % kTsScratchBufs) * 3 * (a.P.cap_cs + a.P.cap_tp + kTsContactCap);
      double* tp = cs + 3 * (size_t)a.P.cap_cs;
      // ---- phase 1, one thread per stored block A_ij (i = r0 + il, j <= i): cs[q] = A v_j; an
      // off-diagonal block also writes A^T v_i to its slot tp[tslot[q]] (grouped by target row)
      for (int q = ct; q < nb; q += kTsConsumers) {
        const unsigned cd = M.code[q];
        const int bl = (int)(cd & 0xffu), jr = (int)((cd >> 8) & 0xffffu);
        const unsigned kind = cd >> 24;
        const double* vj = kind == 2u ? xv + 3 * jr : vt + 3 * jr;
        const VT* A = vals + 9 * q;
        double m[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) m[k] = (double)A[k];  // FP64 arithmetic either way
        const double j0 = vj[0], j1 = vj[1], j2 = vj[2];
        double* c3 = cs + 3 * (int)M.cpos[q];
        c3[0] = fma(m[2], j2, fma(m[1], j1, m[0] * j0));
        c3[1] = fma(m[5], j2, fma(m[4], j1, m[3] * j0));
        c3[2] = fma(m[8], j2, fma(m[7], j1, m[6] * j0));
        if (kind != 0u) {
          const double i0 = vt[3 * bl], i1 = vt[3 * bl + 1], i2 = vt[3 * bl + 2];
          double* t = tp + 3 * (int)M.tslot[q];
          t[0] = fma(m[6], i2, fma(m[3], i1, m[0] * i0));
          t[1] = fma(m[7], i2, fma(m[4], i1, m[1] * i0));
          t[2] = fma(m[8], i2, fma(m[5], i1, m[2] * i0));
        }
      }
      TS_T(6)
      // contact blocks of the tile's rows (one contiguous range of the row-sorted contact BSR): one
      // thread per block, C_s v_col -> cc[s] (the first kTsContactCap of the tile; the rest, rare,
      // are taken by their row thread in phase 2)
      const int* cr = reinterpret_cast<const int*>(S + a.P.o_crp);
      double* cc = tp + 3 * (size_t)a.P.cap_tp;
      const int c0r = crp ? cr[0] : 0;
      const int ncc = crp ? min(cr[R] - c0r, kTsContactCap) : 0;
      for (int e = ct; e < ncc; e += kTsConsumers) {
        const size_t s2 = (size_t)(c0r + e);
        const double* A = a.C.val + 9 * s2;
        const double* vc = a.v + 3 * (size_t)__ldg(a.C.col + s2);
        double m[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) m[k] = __ldg(A + k);
        const double c0 = __ldg(vc), c1 = __ldg(vc + 1), c2 = __ldg(vc + 2);
        cc[3 * e] = fma(m[2], c2, fma(m[1], c1, m[0] * c0));
        cc[3 * e + 1] = fma(m[5], c2, fma(m[4], c1, m[3] * c0));
        cc[3 * e + 2] = fma(m[8], c2, fma(m[7], c1, m[6] * c0));
      }
      bar_consumers();
      TS_T(1)
      // ---- phase 2, fixed-order sums, one thread per owned row il: stored blocks (ascending
      // column), in-tile mirror products (ascending row), contact blocks (ascending column); one
      // thread per out-of-tile target x: its products (ascending block)
      if (ct < R) {
        const int il = ct;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
        sum3(cs, M.rpc[il], M.rpc[il] + M.rle[il], acc0, acc1, acc2);
        sum3(tp, M.mps[il], M.mps[il] + M.mle[il], acc0, acc1, acc2);
        if (crp) {
          const int e0 = cr[il] - c0r, e1 = cr[il + 1] - c0r;
          sum3(cc, e0, min(e1, ncc), acc0, acc1, acc2);
          for (int s2 = c0r + max(e0, ncc); s2 < c0r + e1; ++s2) {
            const double* A = a.C.val + 9 * (size_t)s2;
            const double* vc = a.v + 3 * (size_t)__ldg(a.C.col + s2);
            const double c0 = __ldg(vc), c1 = __ldg(vc + 1), c2 = __ldg(vc + 2);
            acc0 += fma(A[2], c2, fma(A[1], c1, A[0] * c0));
            acc1 += fma(A[5], c2, fma(A[4], c1, A[3] * c0));
            acc2 += fma(A[8], c2, fma(A[7], c1, A[6] * c0));
          }
        }
        double* yr = a.y + 3 * (size_t)(r0 + il);
        yr[0] = acc0;
        yr[1] = acc1;
        yr[2] = acc2;
        if (DOT) dacc += vt[3 * il] * acc0 + vt[3 * il + 1] * acc1 + vt[3 * il + 2] * acc2;
      }
      // partials: consumer threads without a row first (x = ct - R), then the row threads
      for (int x = (ct - R + kTsConsumers) % kTsConsumers; x < nc; x += kTsConsumers) {
        double p0 = 0.0, p1 = 0.0, p2 = 0.0;
        sum3(tp, M.xps[x], M.xps[x] + M.xle[x], p0, p1, p2);
        double* pp = a.part + 3 * (size_t)M.pslot[x];
        pp[0] = p0;
        pp[1] = p1;
        pp[2] = p2;
        if (DOT) dacc += xv[3 * x] * p0 + xv[3 * x + 1] * p1 + xv[3 * x + 2] * p2;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + it % kTsStages);  // this warp is done with the stage
      if (kTsScratchBufs == 1) bar_consumers();            // the next tile's phase 1 reuses cs / tp
      TS_T(2)
    }
  }
#ifdef BAL_TS_TIMING
  if (lane == 0 && (warp == 0 || warp == 1))
    for (int k = 0; k < 8; ++k) atomicAdd(g_ts_timing + 8 * (warp == 1) + k, (unsigned long long)tacc[k]);
#endif
  if (DOT) {
    __shared__ double sh[kTsThreads / 32];
    __shared__ bool last;
    const double bs = block_sum<kTsThreads>(dacc, sh);
    if (tid == 0) {
      a.dpart[blockIdx.x] = bs;
      __threadfence();
      last = (atomicAdd(a.counter, 1u) == (unsigned)G - 1u);
    }
    __syncthreads();
    if (last) {
      __threadfence();
      const bool wx = a.sc->crit == 2;  // criterion (ii) needs ||x_k||: (x,x) partials after the pairs
      double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
      for (int i = tid; i < G; i += kTsThreads) t0 += a.dpart[i];
      for (int i = tid; i < kVecBlocks; i += kTsThreads) {
        t1 += a.upart[2 * i];
        t2 += a.upart[2 * i + 1];
        if (wx) t3 += a.upart[2 * kVecBlocks + i];
      }
      const double delta = block_sum<kTsThreads>(t0, sh);
      const double gam = block_sum<kTsThreads>(t1, sh);
      const double rr = block_sum<kTsThreads>(t2, sh);
      const double xx = wx ? block_sum<kTsThreads>(t3, sh) : 0.0;
      if (tid == 0) {
        cg_scalars(a.sc, a.hist, gam, rr, delta, xx);
        *a.counter = 0u;
      }
    }
  }
}

__global__ void __launch_bounds__(kVecThreads)
k_ts_combine(int n, const int* __restrict__ pin_ptr, const double* __restrict__ part, double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int e0 = pin_ptr[i], e1 = pin_ptr[i + 1];
    if (e0 == e1) continue;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double acc = y[3 * (size_t)i + c];
      for (int e = e0; e < e1; ++e) acc += part[3 * (size_t)e + c];
      y[3 * (size_t)i + c] = acc;
    }
  }
}

namespace {
int ts_cpref() {  // BAL_TS_NO_CPREFETCH=1: no L2 prefetch of the contact ranges (ablation)
  static const int on = getenv("BAL_TS_NO_CPREFETCH") ? 0 : 1;
  return on;
}
template <bool DOT, typename VT>
int ts_grid_t(const TsPlan& P) {
  static int per_sm = -1;
  static size_t smem = 0;
  if (per_sm < 0 || smem != P.smem) {
    CK(cudaFuncSetAttribute(k_spmv_ts<DOT, VT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_ts<DOT, VT>, kTsThreads, P.smem));
    smem = P.smem;
  }
  if (per_sm <= 0) return 0;
  return std::max(1, std::min(per_sm * num_sms(), P.ntiles));
}
template <bool DOT>
int ts_grid(const TsPlan& P) {
  return P.val_bytes == 36 ? ts_grid_t<DOT, float>(P) : ts_grid_t<DOT, double>(P);
}
template <bool DOT>
void ts_launch(int g, cudaStream_t st, const TsArgs& a) {
  if (a.P.val_bytes == 36) k_spmv_ts<DOT, float><<<g, kTsThreads, a.P.smem, st>>>(a);
  else k_spmv_ts<DOT, double><<<g, kTsThreads, a.P.smem, st>>>(a);
}
}  // namespace

int ts_prepare(const TsPlan& P) {  // attributes / occupancy outside any stream capture
  if (P.ntiles <= 0) return 0;
  (void)ts_grid<false>(P);
  return ts_grid<true>(P);
}

bool ts_usable(const Bsr& S) { return S.ts && S.ts->ntiles > 0 && S.r0 == 0 && S.row_end() == S.n; }

void launch_spmv_ts(cudaStream_t st, const Bsr& S, const Bsr& C, const double* v, double* y, double* part,
                    bool combine) {
  const int g = ts_grid<false>(*S.ts);
  if (g <= 0) throw CudaError("k_spmv_ts: no resident CTA (shared memory)");
  TsArgs a{*S.ts, S.ts->val_bytes == 36 ? (const void*)S.val32 : (const void*)S.val, C, v, y, part,
           nullptr, nullptr, nullptr, nullptr, nullptr, ts_cpref()};
#ifdef BAL_TS_TIMING
  unsigned long long z[16] = {0};
  CK(cudaMemcpyToSymbolAsync(g_ts_timing, z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
#endif
  ts_launch<false>(g, st, a);
  CK(cudaGetLastError());
#ifdef BAL_TS_TIMING
  CK(cudaMemcpyFromSymbolAsync(z, g_ts_timing, sizeof(z), 0, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  fprintf(stderr,
          "[ts-timing] kcyc/CTA producer: wait-empty %.1f issue %.1f wait-full %.1f gather %.1f loop %.1f | "
          "consumer w1: wait-full %.1f wait-gath %.1f ph1 %.1f bar %.1f ph2+arrive %.1f loop %.1f\n",
          z[0] / 1e3 / g, z[1] / 1e3 / g, z[2] / 1e3 / g, z[3] / 1e3 / g, z[7] / 1e3 / g, z[12] / 1e3 / g,
          z[13] / 1e3 / g, z[14] / 1e3 / g, z[9] / 1e3 / g, z[10] / 1e3 / g, z[15] / 1e3 / g);
#endif
  if (combine) {
    k_ts_combine<<<kVecBlocks, kVecThreads, 0, st>>>(S.n, S.ts->pin_ptr, part, y);
    CK(cudaGetLastError());
  }
}

void launch_spmv_ts_dot(cudaStream_t st, const Bsr& S, const Bsr& C, const double* u, double* w, double* part,
                        double* dpart, unsigned* counter, PcgScal* sc, const double* upart, double* hist) {
  const int g = ts_grid<true>(*S.ts);
  if (g <= 0) throw CudaError("k_spmv_ts: no resident CTA (shared memory)");
  TsArgs a{*S.ts, S.ts->val_bytes == 36 ? (const void*)S.val32 : (const void*)S.val, C, u, w, part, dpart,
           counter, sc, upart, hist, ts_cpref()};
  ts_launch<true>(g, st, a);
  CK(cudaGetLastError());
}

}  // namespace bal
