// common.cuh -- shared device helpers of libbal (sm_100a, FP64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <stdexcept>
#include <string>

#define BAL_HD __host__ __device__ __forceinline__
#define BAL_D __device__ __forceinline__

namespace bal {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};
struct OomError : std::runtime_error {
  explicit OomError(const std::string& s) : std::runtime_error(s) {}
};
struct NcclError : std::runtime_error {
  explicit NcclError(const std::string& s) : std::runtime_error(s) {}
};

#define CK(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      if (e_ == cudaErrorMemoryAllocation)                                                  \
        throw ::bal::OomError(std::string("CUDA OOM at ") + __FILE__ + ":" +                \
                              std::to_string(__LINE__));                                    \
      throw ::bal::CudaError(std::string(cudaGetErrorString(e_)) + " at " + __FILE__ + ":" + \
                             std::to_string(__LINE__));                                     \
    }                                                                                       \
  } while (0)

// 148 SMs on B200: grid sizes for grid-stride / reduction kernels are multiples of it.
constexpr int kSMs = 148;
// SM count of the current device (MIG / MPS partitions may expose fewer): persistent and
// cooperative grids are sized from it.
inline int num_sms() {
  static int n[64] = {0};
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) return kSMs;
  if (n[d] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0) v = kSMs;
    n[d] = v;
  }
  return n[d];
}
constexpr int kRedBlocks = 4 * kSMs;  // fixed reduction grid -> deterministic partial order
constexpr int kRedThreads = 256;

BAL_D double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
BAL_D double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum (fixed tree): every thread gets the block total.
template <int NT>
BAL_D double block_sum(double v, double* sh /*[NT/32]*/) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (l < NT / 32) ? sh[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}
template <int NT>
BAL_D double block_min(double v, double* sh) {
  v = warp_min(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (l < NT / 32) ? sh[l] : 1.0e300;
    t = warp_min(t);
    if (l == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// 3-vector helpers
struct d3 {
  double x, y, z;
};
BAL_HD d3 mk(double a, double b, double c) { return d3{a, b, c}; }
BAL_HD d3 operator+(d3 a, d3 b) { return d3{a.x + b.x, a.y + b.y, a.z + b.z}; }
BAL_HD d3 operator-(d3 a, d3 b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
BAL_HD d3 operator*(double s, d3 a) { return d3{s * a.x, s * a.y, s * a.z}; }
BAL_HD double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
BAL_HD d3 cross(d3 a, d3 b) {
  return d3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
BAL_HD double comp(d3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
BAL_D d3 ld3(const double* x, int i) { return d3{x[3 * i], x[3 * i + 1], x[3 * i + 2]}; }

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace bal
