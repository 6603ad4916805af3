// partition.cu -- host logic of the vertex-domain partition: contiguous
// block-row ranges balanced by SpMV cost, and the ghost columns a rank must receive per SpMV.  Host
// only (no CUDA calls), so the N > 1 data flow is testable on CPU (tests/test_partition.py, gloo).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/bal.h"

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

}  // extern "C"
