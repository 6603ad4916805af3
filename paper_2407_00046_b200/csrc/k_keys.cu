// k_keys.cu -- 128-bit constraint-key sorting / dedup and the A u A' stencil union
// (SURVEY Q10, Q22, Q28): a constraint is identified by (type, canonical node ids); duplicates
// reached from several primitive pairs count once; A and A' keys merge into one stencil each.
#include <cub/cub.cuh>

#include "geometry.cuh"
#include "keys.h"

namespace bal {

__global__ void k_pack_keys(int n, const int* __restrict__ keys5, unsigned long long* hi, unsigned long long* lo,
                            int* idx, int offset) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Key k;
  k.t = keys5[5 * (size_t)i];
  for (int a = 0; a < 4; ++a) k.n[a] = keys5[5 * (size_t)i + 1 + a];
  hi[offset + i] = key_hi(k);
  lo[offset + i] = key_lo(k);
  idx[offset + i] = offset + i;
}

void KeySorter::sort(cudaStream_t st, int n) {
  // Stable LSD on (hi, lo): pass 1 sorts positions by lo, pass 2 stably by hi.
  hi2.reserve(n);
  lo2.reserve(n);
  idx2.reserve(n);
  if (n <= 0) return;
  size_t t1 = 0, t2 = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, t1, lo.ptr, lo2.ptr, idx.ptr, idx2.ptr, n, 0, 64, st));
  CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, hi2.ptr, hi.ptr, idx2.ptr, idx.ptr, n, 0, 64, st));
  tmp.reserve(std::max(t1, t2));
  CK(cub::DeviceRadixSort::SortPairs(tmp.ptr, t1, lo.ptr, lo2.ptr, idx.ptr, idx2.ptr, n, 0, 64, st));
  gather_u64(st, n, hi.ptr, idx2.ptr, idx_base, hi2.ptr);  // hi in lo-sorted order
  CK(cub::DeviceRadixSort::SortPairs(tmp.ptr, t2, hi2.ptr, hi.ptr, idx2.ptr, idx.ptr, n, 0, 64, st));
  gather_u64(st, n, lo_orig.ptr, idx.ptr, idx_base, lo.ptr);  // lo in final order
}

__global__ void k_gather_u64(int n, const unsigned long long* __restrict__ src, const int* __restrict__ idx, int base,
                             unsigned long long* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  dst[i] = src[idx[i] - base];
}
void gather_u64(cudaStream_t st, int n, const unsigned long long* src, const int* idx, int base,
                unsigned long long* dst) {
  if (n <= 0) return;
  k_gather_u64<<<ceil_div(n, 256), 256, 0, st>>>(n, src, idx, base, dst);
  CK(cudaGetLastError());
}

void KeySorter::prepare(int n) {
  hi.reserve(n);
  lo.reserve(n);
  lo_orig.reserve(n);
  idx.reserve(n);
}

void KeySorter::sort_packed(cudaStream_t st, int n) {
  if (n <= 0) return;
  CK(cudaMemcpyAsync(lo_orig.ptr, lo.ptr, n * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
  sort(st, n);
}

// unique flags over sorted (hi, lo)
__global__ void k_unique_flags(int n, const unsigned long long* hi, const unsigned long long* lo, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (i == 0 || hi[i] != hi[i - 1] || lo[i] != lo[i - 1]) ? 1 : 0;
}
__global__ void k_unique_starts(int n, const int* flag, const int* scan, int* start, int* count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (flag[i]) start[scan[i]] = i;
  if (i == n - 1) {
    start[scan[i] + flag[i]] = n;
    *count = scan[i] + flag[i];
  }
}

int KeySorter::unique(cudaStream_t st, int n) {
  nuniq = 0;
  if (n <= 0) return 0;
  flag.reserve(n);
  scan.reserve(n);
  start.reserve(n + 1);
  cnt.reserve(1);
  k_unique_flags<<<ceil_div(n, 256), 256, 0, st>>>(n, hi.ptr, lo.ptr, flag.ptr);
  size_t t = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, t, flag.ptr, scan.ptr, n, st));
  tmp.reserve(t);
  CK(cub::DeviceScan::ExclusiveSum(tmp.ptr, t, flag.ptr, scan.ptr, n, st));
  k_unique_starts<<<ceil_div(n, 256), 256, 0, st>>>(n, flag.ptr, scan.ptr, start.ptr, cnt.ptr);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&nuniq, cnt.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return nuniq;
}

// ---------------------------------------------------------------- A u A' stencil union
__global__ void k_union_emit(int nu, const int* __restrict__ start, const int* __restrict__ idx,
                             const unsigned long long* __restrict__ hi, const unsigned long long* __restrict__ lo,
                             int nA, const double* __restrict__ ap_mu, const double* __restrict__ ap_s,
                             int* __restrict__ out_keys, double* __restrict__ inA, double* __restrict__ inAp,
                             double* __restrict__ mu, double* __restrict__ s) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nu) return;
  const int b = start[u], e = start[u + 1];
  double fa = 0.0, fap = 0.0, m = 0.0, sv = 0.0;
  for (int j = b; j < e; ++j) {
    const int id = idx[j];
    if (id < nA) {
      fa = 1.0;
    } else {
      fap = 1.0;
      m = ap_mu[id - nA];
      sv = ap_s[id - nA];
    }
  }
  const Key k = key_from(hi[b], lo[b]);
  out_keys[5 * (size_t)u] = k.t;
  for (int a = 0; a < 4; ++a) out_keys[5 * (size_t)u + 1 + a] = k.n[a];
  inA[u] = fa;
  inAp[u] = fap;
  mu[u] = m;
  s[u] = sv;
}

int stencil_union(cudaStream_t st, KeySorter& ks, int nA, const int* keysA, int nAp, const int* keysAp,
                  const double* ap_mu, const double* ap_s, StencilSet& out) {
  const int n = nA + nAp;
  out.n = 0;
  if (n == 0) return 0;
  ks.prepare(n);
  ks.idx_base = 0;
  if (nA) k_pack_keys<<<ceil_div(nA, 256), 256, 0, st>>>(nA, keysA, ks.hi.ptr, ks.lo.ptr, ks.idx.ptr, 0);
  if (nAp) k_pack_keys<<<ceil_div(nAp, 256), 256, 0, st>>>(nAp, keysAp, ks.hi.ptr, ks.lo.ptr, ks.idx.ptr, nA);
  CK(cudaGetLastError());
  ks.sort_packed(st, n);
  const int nu = ks.unique(st, n);
  out.reserve(nu);
  k_union_emit<<<ceil_div(nu, 256), 256, 0, st>>>(nu, ks.start.ptr, ks.idx.ptr, ks.hi.ptr, ks.lo.ptr, nA, ap_mu,
                                                   ap_s, out.keys.ptr, out.inA.ptr, out.inAp.ptr, out.mu.ptr,
                                                   out.s.ptr);
  CK(cudaGetLastError());
  out.n = nu;
  return nu;
}

}  // namespace bal
