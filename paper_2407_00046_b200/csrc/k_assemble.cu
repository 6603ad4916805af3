// k_assemble.cu -- atomic-free assembly of the Newton system.
//
// A = M/h^2 + sum_i S_i^T P(H_i) S_i ("stored separately": a static part
// over the mesh adjacency and a contact part rebuilt every Newton iteration), fixed DOFs ->
// identity rows/columns (App. C; Q23).  Every BSR slot owns a precomputed, fixed-order list
// of (stencil, local block) contributions and sums them itself: no atomics, bitwise
// deterministic.  Static lists are built once at init; contact lists come from a radix sort of
// (row, col) keys every Newton iteration.  The node pass then forms e = grad L, Lambda / e_j /
// group = floor(log10 e_j) (Q17-Q19) and the block-Jacobi inverse.
#include <cub/cub.cuh>

#include "assemble.h"
#include "common.cuh"
#include "kernels.h"

namespace bal {

// decimal literal table 1e-60 .. 1e60 for the exact decade floor (Q19)
__constant__ double c_dec[121];

void init_decades() {
  static bool done = false;
  if (done) return;
  double h[121];
  for (int k = -60; k <= 60; ++k) {
    char buf[16];
    snprintf(buf, sizeof(buf), "1e%d", k);
    h[k + 60] = strtod(buf, nullptr);
  }
  CK(cudaMemcpyToSymbol(c_dec, h, sizeof(h)));
  done = true;
}

BAL_D int floor_log10_exact(double e) {
  int g = (int)floor(log10(e));
  if (g < -60) g = -60;
  if (g > 59) g = 59;
  while (g > -60 && e < c_dec[g + 60]) --g;
  while (g < 59 && e >= c_dec[g + 61]) ++g;
  return g;
}

BAL_D void add_block(double (&acc)[9], const double* __restrict__ blk, bool transpose) {
  if (!transpose) {
#pragma unroll
    for (int t = 0; t < 9; ++t) acc[t] += blk[t];
  } else {
#pragma unroll
    for (int t = 0; t < 9; ++t) acc[t] += blk[3 * (t % 3) + t / 3];
  }
}

// code = stencil*16 + a*4 + b : the (a,b) block of that stencil's P(H)
BAL_D const double* code_block(const double* __restrict__ stage, int code, bool& transpose) {
  const int s = code >> 4, a = (code >> 2) & 3, b = code & 3;
  transpose = a < b;
  const int hi = a > b ? a : b, lo = a > b ? b : a;
  return stage + 90 * (size_t)s + 9 * (hi * (hi + 1) / 2 + lo);
}

__global__ void k_gather_static(int nnzb, const int* __restrict__ slot_row, const int* __restrict__ col,
                                const int* __restrict__ slot_ptr, const int* __restrict__ slot_code,
                                const double* __restrict__ stage, const double* __restrict__ mass, double inv_h2,
                                const uint8_t* __restrict__ fixed, double* __restrict__ val,
                                const int* __restrict__ lpos, double* __restrict__ lval, float* __restrict__ lval32) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nnzb) return;
  const int i = slot_row[s], j = col[s];
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (fixed[i] || fixed[j]) {
    if (i == j) acc[0] = acc[4] = acc[8] = 1.0;
  } else {
    if (i == j) acc[0] = acc[4] = acc[8] = mass[i] * inv_h2;
    for (int c = slot_ptr[s]; c < slot_ptr[s + 1]; ++c) {
      bool tr;
      const double* blk = code_block(stage, slot_code[c], tr);
      add_block(acc, blk, tr);
    }
  }
  double* o = val + 9 * (size_t)s;
#pragma unroll
  for (int t = 0; t < 9; ++t) o[t] = acc[t];
  if (lval) {
    const int lp = lpos[s];
    if (lp >= 0) {
      double* ol = lval + 9 * (size_t)lp;
#pragma unroll
      for (int t = 0; t < 9; ++t) ol[t] = acc[t];
      if (lval32) {  // BAL_FP32_MATRIX: the SpMV's stored blocks rounded to FP32
        float* o32 = lval32 + 9 * (size_t)lp;
#pragma unroll
        for (int t = 0; t < 9; ++t) o32[t] = (float)acc[t];
      }
    }
  }
}

// contact slots: contributions are the sorted entries [start[s], start[s+1])
__global__ void k_gather_contact(int nslots, const unsigned long long* __restrict__ keys,
                                 const int* __restrict__ codes, const int* __restrict__ start,
                                 const double* __restrict__ stage, int* __restrict__ ccol, double* __restrict__ cval) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslots) return;
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  const int b = start[s], e = start[s + 1];
  for (int c = b; c < e; ++c) {
    bool tr;
    const double* blk = code_block(stage, codes[c], tr);
    add_block(acc, blk, tr);
  }
  ccol[s] = (int)(keys[b] & 0xffffffffull);
  double* o = cval + 9 * (size_t)s;
#pragma unroll
  for (int t = 0; t < 9; ++t) o[t] = acc[t];
}

// emit (row,col) keys for every block of every contact/friction stencil with both nodes free
__global__ void k_contact_entries(int ns, const int* __restrict__ nodes, const uint8_t* __restrict__ fixed,
                                  unsigned long long* __restrict__ keys, int* __restrict__ codes) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= ns) return;
  int nd[4];
  for (int a = 0; a < 4; ++a) nd[a] = nodes[4 * (size_t)s + a];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      const size_t o = 16 * (size_t)s + 4 * a + b;
      const bool ok = nd[a] >= 0 && nd[b] >= 0 && !fixed[nd[a]] && !fixed[nd[b]];
      keys[o] = ok ? (((unsigned long long)nd[a] << 32) | (unsigned)nd[b]) : ~0ull;
      codes[o] = s * 16 + 4 * a + b;
    }
}

__global__ void k_slot_flags(int m, const unsigned long long* __restrict__ keys, int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const unsigned long long k = keys[i];
  flag[i] = (k != ~0ull && (i == 0 || keys[i - 1] != k)) ? 1 : 0;
}

__global__ void k_slot_starts(int m, const unsigned long long* __restrict__ keys, const int* __restrict__ flag,
                              const int* __restrict__ scan, int* __restrict__ start, int* __restrict__ nvalid_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (flag[i]) start[scan[i]] = i;
  const bool valid = keys[i] != ~0ull;
  const bool next_invalid = (i + 1 == m) || keys[i + 1] == ~0ull;
  if (valid && next_invalid) {
    start[scan[i] + flag[i]] = i + 1;  // sentinel end
    *nvalid_out = scan[i] + flag[i];
  }
}

// contact CSR row pointers: row_ptr[r] = first slot with row >= r
__global__ void k_contact_rowptr(int n, int nslots, const unsigned long long* __restrict__ keys,
                                 const int* __restrict__ start, int* __restrict__ row_ptr) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > n) return;
  int lo = 0, hi = nslots;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const int row = (int)(keys[start[mid]] >> 32);
    if (row < r) lo = mid + 1;
    else hi = mid;
  }
  row_ptr[r] = lo;
}

__global__ void k_count_rows(int n, const int* __restrict__ row_ptr, int* cnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int ne = (r < n && row_ptr[r + 1] > row_ptr[r]) ? 1 : 0;
  const int s = __syncthreads_count(ne);
  if (threadIdx.x == 0 && s) atomicAdd(cnt, s);
}

// per node: gradient, Lambda -> e_j, group, diagonal block inverse
__global__ void k_node_finalize(int n, const double* __restrict__ x, const double* __restrict__ y,
                                const double* __restrict__ mass, double inv_h2, const uint8_t* __restrict__ fixed,
                                const int* __restrict__ diag_pos, const int* __restrict__ slot_ptr,
                                const int* __restrict__ slot_code, const double* __restrict__ grad_e,
                                const double* __restrict__ lbar_e, const double* __restrict__ sval,
                                const int* __restrict__ c_row_ptr, const int* __restrict__ c_col,
                                const double* __restrict__ c_val, const int* __restrict__ c_start,
                                const int* __restrict__ c_codes, const double* __restrict__ grad_c,
                                const double* __restrict__ lbar_c, double* __restrict__ grad,
                                double* __restrict__ e_node, int* __restrict__ group, double* __restrict__ dinv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double m2 = mass[i] * inv_h2;
  double g0 = m2 * (x[3 * (size_t)i] - y[3 * (size_t)i]);
  double g1 = m2 * (x[3 * (size_t)i + 1] - y[3 * (size_t)i + 1]);
  double g2 = m2 * (x[3 * (size_t)i + 2] - y[3 * (size_t)i + 2]);
  double L = m2;
  const int ds = diag_pos[i];
  for (int c = slot_ptr[ds]; c < slot_ptr[ds + 1]; ++c) {
    const int code = slot_code[c];
    const int e = code >> 4, a = (code >> 2) & 3;
    g0 += grad_e[12 * (size_t)e + 3 * a];
    g1 += grad_e[12 * (size_t)e + 3 * a + 1];
    g2 += grad_e[12 * (size_t)e + 3 * a + 2];
    L += lbar_e[e];
  }
  double D[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) D[t] = sval[9 * (size_t)ds + t];
  if (c_row_ptr != nullptr) {
    for (int s = c_row_ptr[i]; s < c_row_ptr[i + 1]; ++s) {
      if (c_col[s] != i) continue;
#pragma unroll
      for (int t = 0; t < 9; ++t) D[t] += c_val[9 * (size_t)s + t];
      for (int c = c_start[s]; c < c_start[s + 1]; ++c) {
        const int code = c_codes[c];
        const int st = code >> 4, a = (code >> 2) & 3;
        g0 += grad_c[12 * (size_t)st + 3 * a];
        g1 += grad_c[12 * (size_t)st + 3 * a + 1];
        g2 += grad_c[12 * (size_t)st + 3 * a + 2];
        L += lbar_c[st];
      }
    }
  }
  double* di = dinv + 6 * (size_t)i;
  if (fixed[i]) {
    grad[3 * (size_t)i] = grad[3 * (size_t)i + 1] = grad[3 * (size_t)i + 2] = 0.0;
    e_node[i] = 3.0 * L;
    group[i] = INT_MIN;
    di[0] = 1.0; di[1] = 0.0; di[2] = 0.0; di[3] = 1.0; di[4] = 0.0; di[5] = 1.0;
    return;
  }
  grad[3 * (size_t)i] = g0;
  grad[3 * (size_t)i + 1] = g1;
  grad[3 * (size_t)i + 2] = g2;
  const double e = (L + L) + L;
  e_node[i] = e;
  group[i] = floor_log10_exact(e);
  // symmetric 3x3 inverse via cofactors (D symmetric by construction)
  const double a = D[0], b = D[1], c = D[2], d = D[4], f = D[5], k = D[8];
  const double A0 = d * k - f * f, A1 = c * f - b * k, A2 = b * f - c * d;
  const double det = a * A0 + b * A1 + c * A2;
  const double id = 1.0 / det;
  di[0] = A0 * id;
  di[1] = A1 * id;
  di[2] = A2 * id;
  di[3] = (a * k - c * c) * id;
  di[4] = (b * c - a * f) * id;
  di[5] = (a * d - b * b) * id;
}

// ---------------------------------------------------------------------------- host side
void gather_static(cudaStream_t st, const StaticPattern& sp, const double* stage, const double* mass,
                   double inv_h2, const uint8_t* fixed, double* val, double* lval, float* lval32) {
  k_gather_static<<<ceil_div(sp.nnzb, 256), 256, 0, st>>>(sp.nnzb, sp.slot_row, sp.col, sp.slot_ptr, sp.slot_code,
                                                           stage, mass, inv_h2, fixed, val, sp.lpos, lval, lval32);
  CK(cudaGetLastError());
}

int build_contact_pattern(cudaStream_t st, ContactWork& w, int ns, const int* nodes, const uint8_t* fixed, int n,
                          const double* stage) {
  w.nslots = 0;
  w.nrows = 0;
  if (ns <= 0) return 0;
  const int m = 16 * ns;
  w.keys.reserve(m);
  w.keys_alt.reserve(m);
  w.codes.reserve(m);
  w.codes_alt.reserve(m);
  w.flag.reserve(m + 1);
  w.scan.reserve(m + 1);
  w.start.reserve(m + 2);
  k_contact_entries<<<ceil_div(ns, 128), 128, 0, st>>>(ns, nodes, fixed, w.keys.ptr, w.codes.ptr);
  CK(cudaGetLastError());
  size_t tmp = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, w.keys.ptr, w.keys_alt.ptr, w.codes.ptr, w.codes_alt.ptr, m, 0,
                                     64, st));
  w.tmp.reserve(tmp);
  CK(cub::DeviceRadixSort::SortPairs(w.tmp.ptr, tmp, w.keys.ptr, w.keys_alt.ptr, w.codes.ptr, w.codes_alt.ptr, m, 0,
                                     64, st));
  k_slot_flags<<<ceil_div(m, 256), 256, 0, st>>>(m, w.keys_alt.ptr, w.flag.ptr);
  size_t tmp2 = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, w.flag.ptr, w.scan.ptr, m, st));
  w.tmp.reserve(tmp2);
  CK(cub::DeviceScan::ExclusiveSum(w.tmp.ptr, tmp2, w.flag.ptr, w.scan.ptr, m, st));
  w.nvalid.reserve(1);
  CK(cudaMemsetAsync(w.nvalid.ptr, 0, sizeof(int), st));
  k_slot_starts<<<ceil_div(m, 256), 256, 0, st>>>(m, w.keys_alt.ptr, w.flag.ptr, w.scan.ptr, w.start.ptr,
                                                   w.nvalid.ptr);
  CK(cudaGetLastError());
  int nslots = 0;
  CK(cudaMemcpyAsync(&nslots, w.nvalid.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  w.nslots = nslots;
  w.row_ptr.reserve(n + 1);
  w.col.reserve(std::max(nslots, 1));
  w.val.reserve(9 * (size_t)std::max(nslots, 1));
  k_contact_rowptr<<<ceil_div(n + 1, 256), 256, 0, st>>>(n, nslots, w.keys_alt.ptr, w.start.ptr, w.row_ptr.ptr);
  if (nslots > 0)
    k_gather_contact<<<ceil_div(nslots, 256), 256, 0, st>>>(nslots, w.keys_alt.ptr, w.codes_alt.ptr, w.start.ptr,
                                                             stage, w.col.ptr, w.val.ptr);
  CK(cudaMemsetAsync(w.nvalid.ptr, 0, sizeof(int), st));
  k_count_rows<<<ceil_div(n, 256), 256, 0, st>>>(n, w.row_ptr.ptr, w.nvalid.ptr);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&w.nrows, w.nvalid.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  return nslots;
}

void node_finalize(cudaStream_t st, int n, const double* x, const double* y, const double* mass, double inv_h2,
                   const uint8_t* fixed, const StaticPattern& sp, const double* grad_e, const double* lbar_e,
                   const double* sval, const ContactWork* cw, const double* grad_c, const double* lbar_c,
                   double* grad, double* e_node, int* group, double* dinv) {
  init_decades();
  const bool hc = cw && cw->nslots > 0;
  k_node_finalize<<<ceil_div(n, 256), 256, 0, st>>>(
      n, x, y, mass, inv_h2, fixed, sp.diag_pos, sp.slot_ptr, sp.slot_code, grad_e, lbar_e, sval,
      hc ? cw->row_ptr.ptr : nullptr, hc ? cw->col.ptr : nullptr, hc ? cw->val.ptr : nullptr,
      hc ? cw->start.ptr : nullptr, hc ? cw->codes_alt.ptr : nullptr, grad_c, lbar_c, grad, e_node, group, dinv);
  CK(cudaGetLastError());
}

}  // namespace bal
