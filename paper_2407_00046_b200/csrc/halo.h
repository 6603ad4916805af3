// halo.h -- pack / unpack of the SpMV halo exchange: one routine compiled for the
// host (bal_halo_pack / bal_halo_unpack, CPU tests) and the device (pcg_dist.cu kernels).
#pragma once
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace bal {

// entry k of the halo buffer <-> node idx[k] of a [3N] vector (3 doubles per node)
BAL_HD void halo_pack_entry(int k, const int32_t* idx, const double* v, double* buf) {
  const size_t s = 3 * (size_t)idx[k];
  buf[3 * (size_t)k] = v[s];
  buf[3 * (size_t)k + 1] = v[s + 1];
  buf[3 * (size_t)k + 2] = v[s + 2];
}
BAL_HD void halo_unpack_entry(int k, const int32_t* idx, const double* buf, double* v) {
  const size_t s = 3 * (size_t)idx[k];
  v[s] = buf[3 * (size_t)k];
  v[s + 1] = buf[3 * (size_t)k + 1];
  v[s + 2] = buf[3 * (size_t)k + 2];
}

// Boundary-only halo of one rank: per peer m, send_idx[send_ptr[m] .. send_ptr[m+1]) = owned rows
// whose values m needs, recv_idx[recv_ptr[m] .. recv_ptr[m+1]) = ghost rows owned by m (ascending).
struct HaloPlan {
  std::vector<int32_t> send_ptr, send_idx, recv_ptr, recv_idx;
};

// Builds the plan of `rank` from one or two symmetric block patterns (the static mesh adjacency
// and, optionally, this Newton iteration's contact pattern); bounds[world+1] = row partition.
void halo_plan_build(int n, const int32_t* rp, const int32_t* col, const int32_t* rp2, const int32_t* col2, int world,
                     const int32_t* bounds, int rank, HaloPlan& out);

}  // namespace bal
