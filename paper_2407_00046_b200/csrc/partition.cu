// partition.cu -- host logic of the vertex-domain partition: contiguous
// block-row ranges balanced by SpMV cost, and the ghost columns a rank must receive per SpMV.  Host
// only (no CUDA calls), so the N > 1 data flow is testable on CPU (tests/test_partition.py, gloo).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/bal.h"
#include "halo.h"

namespace bal {

void halo_plan_build(int n, const int32_t* rp, const int32_t* col, const int32_t* rp2, const int32_t* col2, int world,
                     const int32_t* bounds, int rank, HaloPlan& out) {
  const int r0 = bounds[rank], r1 = bounds[rank + 1];
  auto owner = [&](int j) { return (int)(std::upper_bound(bounds, bounds + world + 1, j) - bounds) - 1; };
  std::vector<std::vector<int32_t>> snd(world), rcv(world);
  std::vector<int32_t> last(world, -1);
  auto visit = [&](int i, int j) {
    if (j >= r0 && j < r1) return;
    const int m = owner(j);
    if (last[m] != i) {  // row i (owned) is needed by rank m: rows visited in ascending order
      snd[m].push_back(i);
      last[m] = i;
    }
    rcv[m].push_back(j);
  };
  for (int i = r0; i < r1; ++i) {
    for (int s = rp[i]; s < rp[i + 1]; ++s) visit(i, col[s]);
    if (rp2)
      for (int s = rp2[i]; s < rp2[i + 1]; ++s) visit(i, col2[s]);
  }
  out.send_ptr.assign(world + 1, 0);
  out.recv_ptr.assign(world + 1, 0);
  out.send_idx.clear();
  out.recv_idx.clear();
  for (int m = 0; m < world; ++m) {
    std::sort(rcv[m].begin(), rcv[m].end());
    rcv[m].erase(std::unique(rcv[m].begin(), rcv[m].end()), rcv[m].end());
    out.send_idx.insert(out.send_idx.end(), snd[m].begin(), snd[m].end());
    out.recv_idx.insert(out.recv_idx.end(), rcv[m].begin(), rcv[m].end());
    out.send_ptr[m + 1] = (int32_t)out.send_idx.size();
    out.recv_ptr[m + 1] = (int32_t)out.recv_idx.size();
  }
}

}  // namespace bal

extern "C" {

bal_status bal_partition_rows(int32_t n, const int64_t* row_cost, int32_t world, int32_t* bounds) {
  if (n < 0 || world <= 0 || !bounds || (n > 0 && !row_cost)) return BAL_E_INVALID_ARG;
  // prefix sums of the cost; rank k takes the rows whose prefix midpoint falls in [k/W, (k+1)/W)
  std::vector<long double> pre(n + 1, 0.0L);
  for (int32_t i = 0; i < n; ++i) {
    if (row_cost[i] < 0) return BAL_E_INVALID_ARG;
    pre[i + 1] = pre[i] + (long double)row_cost[i];
  }
  const long double tot = pre[n];
  bounds[0] = 0;
  for (int32_t k = 1; k < world; ++k) {
    const long double target = tot * k / world;
    // first row i with pre[i] >= target (balanced split point), monotone in k
    int32_t i = (int32_t)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
    if (tot == 0.0L) i = (int32_t)((int64_t)n * k / world);
    bounds[k] = std::max(bounds[k - 1], std::min(i, n));
  }
  bounds[world] = n;
  return BAL_OK;
}

int32_t bal_ghost_columns(int32_t n, const int32_t* row_ptr, const int32_t* col, int32_t r0, int32_t r1,
                          int32_t* out, int32_t cap) {
  if (n < 0 || !row_ptr || r0 < 0 || r1 < r0 || r1 > n || cap < 0) return BAL_E_INVALID_ARG;
  std::vector<int32_t> g;
  for (int32_t i = r0; i < r1; ++i)
    for (int32_t s = row_ptr[i]; s < row_ptr[i + 1]; ++s) {
      const int32_t j = col[s];
      if (j < 0 || j >= n) return BAL_E_INVALID_ARG;
      if (j < r0 || j >= r1) g.push_back(j);
    }
  std::sort(g.begin(), g.end());
  g.erase(std::unique(g.begin(), g.end()), g.end());
  const int32_t m = (int32_t)g.size();
  if (out) std::copy(g.begin(), g.begin() + std::min(m, cap), out);
  return m;
}

int32_t bal_halo_plan(int32_t n, const int32_t* row_ptr, const int32_t* col, int32_t world, const int32_t* bounds,
                      int32_t rank, int32_t* send_ptr, int32_t* send_idx, int32_t* recv_ptr, int32_t* recv_idx,
                      int32_t cap) {
  if (n < 0 || !row_ptr || (row_ptr[n] > 0 && !col) || world <= 0 || !bounds || rank < 0 || rank >= world ||
      cap < 0 || !send_ptr || !recv_ptr)
    return BAL_E_INVALID_ARG;
  if (bounds[0] != 0 || bounds[world] != n) return BAL_E_INVALID_ARG;
  for (int32_t k = 0; k < world; ++k)
    if (bounds[k + 1] < bounds[k]) return BAL_E_INVALID_ARG;
  for (int32_t s = 0; s < row_ptr[n]; ++s)
    if (col[s] < 0 || col[s] >= n) return BAL_E_INVALID_ARG;
  bal::HaloPlan p;
  bal::halo_plan_build(n, row_ptr, col, nullptr, nullptr, world, bounds, rank, p);
  std::copy(p.send_ptr.begin(), p.send_ptr.end(), send_ptr);
  std::copy(p.recv_ptr.begin(), p.recv_ptr.end(), recv_ptr);
  if (send_idx) std::copy(p.send_idx.begin(), p.send_idx.begin() + std::min<size_t>(cap, p.send_idx.size()), send_idx);
  if (recv_idx) std::copy(p.recv_idx.begin(), p.recv_idx.begin() + std::min<size_t>(cap, p.recv_idx.size()), recv_idx);
  return (int32_t)std::max(p.send_idx.size(), p.recv_idx.size());
}

bal_status bal_halo_pack(int32_t count, const int32_t* idx, const double* v, double* buf) {
  if (count < 0 || (count > 0 && (!idx || !v || !buf))) return BAL_E_INVALID_ARG;
  for (int32_t k = 0; k < count; ++k) bal::halo_pack_entry(k, idx, v, buf);
  return BAL_OK;
}

bal_status bal_halo_unpack(int32_t count, const int32_t* idx, const double* buf, double* v) {
  if (count < 0 || (count > 0 && (!idx || !v || !buf))) return BAL_E_INVALID_ARG;
  for (int32_t k = 0; k < count; ++k) bal::halo_unpack_entry(k, idx, buf, v);
  return BAL_OK;
}

}  // extern "C"
