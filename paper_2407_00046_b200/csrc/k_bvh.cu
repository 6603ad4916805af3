// k_bvh.cu -- linear BVH broad phase (§5.3): two trees (surface triangles, surface
// edges), 64-bit keys = 30-bit Morton code of the box centroid << 32 | primitive index (the
// paper's "32 bits for the Morton code and an additional 32 bits for safety"), radix sort, Karras
// binary radix tree, bottom-up AABB refit where each internal node is finalised by the second
// child to arrive (the paper's two-visit gate, fig:atomicCAS).  Queries are stackless-per-thread
// stack traversals emitting candidate pairs; the broad phase is result-neutral (any sound
// superset gives the same constraint set and TOI).
#include <cub/cub.cuh>

#include "bvh.h"

namespace bal {

BAL_D void prim_box(int kind, int i, const int* __restrict__ prims, const double* __restrict__ xa,
                    const double* __restrict__ xb, double h, double lo[3], double hi[3]) {
  const int k = kind;  // nodes per primitive: 1 vertex, 2 edge, 3 triangle
  for (int c = 0; c < 3; ++c) {
    lo[c] = INFINITY;
    hi[c] = -INFINITY;
  }
  for (int a = 0; a < k; ++a) {
    const int n = prims[(size_t)k * i + a];
    for (int c = 0; c < 3; ++c) {
      const double va = xa[3 * (size_t)n + c], vb = xb[3 * (size_t)n + c];
      lo[c] = fmin(lo[c], fmin(va, vb));
      hi[c] = fmax(hi[c], fmax(va, vb));
    }
  }
  for (int c = 0; c < 3; ++c) {
    lo[c] -= h;
    hi[c] += h;
  }
}

__global__ void k_prim_boxes(int n, int kind, const int* prims, const double* xa, const double* xb, double h,
                             double* lo, double* hi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double l[3], u[3];
  prim_box(kind, i, prims, xa, xb, h, l, u);
  for (int c = 0; c < 3; ++c) {
    lo[3 * (size_t)i + c] = l[c];
    hi[3 * (size_t)i + c] = u[c];
  }
}

__global__ void k_bounds(int n, const double* lo, const double* hi, double* part) {
  __shared__ double sh[kRedThreads / 32];
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int c = 0; c < 3; ++c) {
      const double m = 0.5 * (lo[3 * (size_t)i + c] + hi[3 * (size_t)i + c]);
      mn[c] = fmin(mn[c], m);
      mx[c] = fmax(mx[c], m);
    }
  for (int c = 0; c < 3; ++c) {
    const double a = block_min<kRedThreads>(mn[c], sh);
    const double b = -block_min<kRedThreads>(-mx[c], sh);
    if (threadIdx.x == 0) {
      part[6 * blockIdx.x + c] = a;
      part[6 * blockIdx.x + 3 + c] = b;
    }
  }
}
__global__ void __launch_bounds__(kRedThreads) k_bounds_finish(int np, const double* part, double* out) {
  __shared__ double sh[kRedThreads / 32];
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int b = threadIdx.x; b < np; b += blockDim.x)
    for (int c = 0; c < 3; ++c) {
      mn[c] = fmin(mn[c], part[6 * b + c]);
      mx[c] = fmax(mx[c], part[6 * b + 3 + c]);
    }
  for (int c = 0; c < 3; ++c) {
    const double a = block_min<kRedThreads>(mn[c], sh);
    const double z = -block_min<kRedThreads>(-mx[c], sh);
    if (threadIdx.x == 0) {
      out[c] = a;
      out[3 + c] = z;
    }
  }
}

BAL_D unsigned expand_bits(unsigned v) {
  v = (v * 0x00010001u) & 0xFF0000FFu;
  v = (v * 0x00000101u) & 0x0F00F00Fu;
  v = (v * 0x00000011u) & 0xC30C30C3u;
  v = (v * 0x00000005u) & 0x49249249u;
  return v;
}

__global__ void k_morton(int n, const double* lo, const double* hi, const double* bounds,
                         unsigned long long* keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned q[3];
  for (int c = 0; c < 3; ++c) {
    const double m = 0.5 * (lo[3 * (size_t)i + c] + hi[3 * (size_t)i + c]);
    const double ext = bounds[3 + c] - bounds[c];
    double t = ext > 0 ? (m - bounds[c]) / ext : 0.5;
    t = fmin(fmax(t, 0.0), 1.0);
    q[c] = (unsigned)fmin(t * 1024.0, 1023.0);
  }
  const unsigned code = (expand_bits(q[0]) << 2) | (expand_bits(q[1]) << 1) | expand_bits(q[2]);
  keys[i] = ((unsigned long long)code << 32) | (unsigned)i;
}

BAL_D int delta(const unsigned long long* k, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  return __clzll(k[i] ^ k[j]);
}

// Karras 2012: internal nodes 0..n-2, leaves n-1 .. 2n-2 (leaf l <-> sorted position l)
__global__ void k_radix_tree(int n, const unsigned long long* __restrict__ k, int* left, int* right, int* parent) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  const int d = (delta(k, n, i, i + 1) - delta(k, n, i, i - 1)) >= 0 ? 1 : -1;
  const int dmin = delta(k, n, i, i - d);
  int lmax = 2;
  while (delta(k, n, i, i + lmax * d) > dmin) lmax *= 2;
  int l = 0;
  for (int t = lmax / 2; t >= 1; t /= 2)
    if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
  const int j = i + l * d;
  const int dnode = delta(k, n, i, j);
  int s = 0, t = l;
  do {
    t = (t + 1) >> 1;
    if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
  } while (t > 1);
  const int gamma = i + s * d + min(d, 0);
  const int lc = (min(i, j) == gamma) ? (n - 1 + gamma) : gamma;
  const int rc = (max(i, j) == gamma + 1) ? (n - 1 + gamma + 1) : gamma + 1;
  left[i] = lc;
  right[i] = rc;
  parent[lc] = i;
  parent[rc] = i;
  if (i == 0) parent[0] = -1;
}

__global__ void k_leaf_boxes(int n, const unsigned long long* __restrict__ k, const double* lo, const double* hi,
                             double* nlo, double* nhi, int* leaf_prim) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= n) return;
  const int p = (int)(k[l] & 0xffffffffull);
  const int node = n - 1 + l;
  leaf_prim[l] = p;
  for (int c = 0; c < 3; ++c) {
    nlo[3 * (size_t)node + c] = lo[3 * (size_t)p + c];
    nhi[3 * (size_t)node + c] = hi[3 * (size_t)p + c];
  }
}

// bottom-up refit: the second child to arrive finalises the parent (two-visit gate)
__global__ void k_refit(int n, const int* __restrict__ left, const int* __restrict__ right,
                        const int* __restrict__ parent, unsigned* visits, double* nlo, double* nhi) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= n) return;
  int node = parent[n - 1 + l];
  while (node >= 0) {
    __threadfence();
    if (atomicAdd(visits + node, 1u) == 0u) return;  // first visitor: the sibling will finish
    const int a = left[node], b = right[node];
    for (int c = 0; c < 3; ++c) {
      nlo[3 * (size_t)node + c] = fmin(__ldcg(nlo + 3 * (size_t)a + c), __ldcg(nlo + 3 * (size_t)b + c));
      nhi[3 * (size_t)node + c] = fmax(__ldcg(nhi + 3 * (size_t)a + c), __ldcg(nhi + 3 * (size_t)b + c));
    }
    node = parent[node];
  }
}

void Lbvh::build(cudaStream_t st, int n_, int kind, const int* prims, const double* xa, const double* xb,
                 double h) {
  n = n_;
  if (n <= 0) return;
  lo.reserve(3 * (size_t)n);
  hi.reserve(3 * (size_t)n);
  keys.reserve(n);
  keys2.reserve(n);
  const int nn = 2 * n - 1;
  nlo.reserve(3 * (size_t)nn);
  nhi.reserve(3 * (size_t)nn);
  left.reserve(std::max(n - 1, 1));
  right.reserve(std::max(n - 1, 1));
  parent.reserve(nn);
  visits.reserve(std::max(n - 1, 1));
  leaf_prim.reserve(n);
  part.reserve(6 * kRedBlocks + 6);
  k_prim_boxes<<<ceil_div(n, 256), 256, 0, st>>>(n, kind, prims, xa, xb, h, lo.ptr, hi.ptr);
  k_bounds<<<kRedBlocks, kRedThreads, 0, st>>>(n, lo.ptr, hi.ptr, part.ptr);
  k_bounds_finish<<<1, kRedThreads, 0, st>>>(kRedBlocks, part.ptr, part.ptr + 6 * kRedBlocks);
  k_morton<<<ceil_div(n, 256), 256, 0, st>>>(n, lo.ptr, hi.ptr, part.ptr + 6 * kRedBlocks, keys.ptr);
  size_t t = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, t, keys.ptr, keys2.ptr, n, 0, 64, st));
  tmp.reserve(t);
  CK(cub::DeviceRadixSort::SortKeys(tmp.ptr, t, keys.ptr, keys2.ptr, n, 0, 64, st));
  if (n > 1) k_radix_tree<<<ceil_div(n - 1, 256), 256, 0, st>>>(n, keys2.ptr, left.ptr, right.ptr, parent.ptr);
  else CK(cudaMemsetAsync(parent.ptr, 0xff, sizeof(int), st));
  k_leaf_boxes<<<ceil_div(n, 256), 256, 0, st>>>(n, keys2.ptr, lo.ptr, hi.ptr, nlo.ptr, nhi.ptr, leaf_prim.ptr);
  if (n > 1) {
    CK(cudaMemsetAsync(visits.ptr, 0, sizeof(unsigned) * (n - 1), st));
    k_refit<<<ceil_div(n, 256), 256, 0, st>>>(n, left.ptr, right.ptr, parent.ptr, visits.ptr, nlo.ptr, nhi.ptr);
  }
  CK(cudaGetLastError());
}

// ------------------------------------------------------------------------------- queries
BAL_D bool overlap(const double ql[3], const double qh[3], const double* __restrict__ nlo,
                   const double* __restrict__ nhi, int node) {
  for (int c = 0; c < 3; ++c)
    if (ql[c] > nhi[3 * (size_t)node + c] || nlo[3 * (size_t)node + c] > qh[c]) return false;
  return true;
}

// mode 0: vertex queries vs triangle tree -> PT pairs (p, a, b, c)
// mode 1: edge queries vs edge tree -> EE pairs (edge q < edge prim)
__global__ void k_query(int nq, int mode, const int* __restrict__ qprims, const int* __restrict__ tprims, int nt,
                        const double* __restrict__ xa, const double* __restrict__ xb, double h,
                        const double* __restrict__ nlo, const double* __restrict__ nhi, const int* __restrict__ left,
                        const int* __restrict__ right, const int* __restrict__ leaf_prim,
                        const uint8_t* __restrict__ fixed, int4* out, int* count, int cap) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const int qk = mode == 0 ? 1 : 2;
  double ql[3], qh[3];
  prim_box(qk, q, qprims, xa, xb, h, ql, qh);
  int qn[2];
  qn[0] = qprims[(size_t)qk * q];
  qn[1] = mode == 1 ? qprims[(size_t)qk * q + 1] : -1;
  const bool qfixed = fixed[qn[0]] && (mode == 0 || fixed[qn[1]]);
  int stack[128];
  int sp = 0;
  stack[sp++] = (nt == 1) ? 0 : 0;
  const bool single = (nt == 1);
  while (sp > 0) {
    const int node = stack[--sp];
    const int nid = single ? 0 : node;  // node index into nlo/nhi (leaf 0 is node 0 when nt == 1)
    if (!overlap(ql, qh, nlo, nhi, nid)) continue;
    const bool is_leaf = single || node >= nt - 1;
    if (!is_leaf) {
      if (sp < 126) {
        stack[sp++] = left[node];
        stack[sp++] = right[node];
      }
      continue;
    }
    const int p = single ? leaf_prim[0] : leaf_prim[node - (nt - 1)];
    int4 pr;
    if (mode == 0) {
      const int a = tprims[3 * (size_t)p], b = tprims[3 * (size_t)p + 1], c = tprims[3 * (size_t)p + 2];
      if (qn[0] == a || qn[0] == b || qn[0] == c) continue;
      if (qfixed && fixed[a] && fixed[b] && fixed[c]) continue;
      pr = make_int4(qn[0], a, b, c);
    } else {
      if (p <= q) continue;
      const int a = tprims[2 * (size_t)p], b = tprims[2 * (size_t)p + 1];
      if (a == qn[0] || a == qn[1] || b == qn[0] || b == qn[1]) continue;
      if (qfixed && fixed[a] && fixed[b]) continue;
      pr = make_int4(qn[0], qn[1], a, b);
    }
    const int slot = atomicAdd(count, 1);
    if (slot < cap) out[slot] = pr;
  }
}

int query_pairs(cudaStream_t st, Lbvh& tree, int mode, int nq, const int* qprims, const int* tprims,
                const double* xa, const double* xb, double h, const uint8_t* fixed, DevBuf<int4>& out,
                DevBuf<int>& cnt) {
  if (nq <= 0 || tree.n <= 0) return 0;
  cnt.reserve(1);
  if (out.cap < 1024) out.reserve(1024);
  for (int attempt = 0; attempt < 4; ++attempt) {
    CK(cudaMemsetAsync(cnt.ptr, 0, sizeof(int), st));
    const int cap = (int)std::min<size_t>(out.cap, (size_t)INT32_MAX);
    k_query<<<ceil_div(nq, 128), 128, 0, st>>>(nq, mode, qprims, tprims, tree.n, xa, xb, h, tree.nlo.ptr,
                                               tree.nhi.ptr, tree.left.ptr, tree.right.ptr, tree.leaf_prim.ptr, fixed,
                                               out.ptr, cnt.ptr, cap);
    CK(cudaGetLastError());
    int c = 0;
    CK(cudaMemcpyAsync(&c, cnt.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (c <= cap) return c;
    out.reserve((size_t)c);
  }
  throw CudaError("broad phase: candidate buffer did not converge");
}

}  // namespace bal
