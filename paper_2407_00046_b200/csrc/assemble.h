// assemble.h -- device buffers and the assembly data structures shared by the host code.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace bal {

// Growable device buffer (never shrinks; contents not preserved on growth).
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
  void reserve(size_t n) {
    if (n <= cap && ptr) return;
    release();
    size_t c = std::max<size_t>(n, 1);
    c = c + c / 4;  // headroom for per-iteration growth
    CK(cudaMalloc(&ptr, c * sizeof(T)));
    cap = c;
  }
  void upload(const T* h, size_t n, cudaStream_t st) {
    reserve(n);
    // h may be an empty vector's data() (nullptr) with n = 1 (minimum-size buffers): reserve only
    if (n && h) CK(cudaMemcpyAsync(ptr, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
  }
};

// Static (mesh adjacency) full BSR pattern + per-slot elastic contribution lists.
struct StaticPattern {
  int n = 0, nnzb = 0;
  int* row_ptr = nullptr;    // [n+1]
  int* col = nullptr;        // [nnzb]
  int* slot_row = nullptr;   // [nnzb]
  int* diag_pos = nullptr;   // [n]
  int* slot_ptr = nullptr;   // [nnzb+1]
  int* slot_code = nullptr;  // [16 T] tet*16 + a*4 + b
  // symmetric copy for the SpMV (kernels.h Bsr): lower + diagonal slots in their own CSR
  int nl = 0, nu = 0;
  int tile_cap_full = 0;  // max full-BSR blocks of an SpMV tile (staged-full mode)
  int* lpos = nullptr;       // [nnzb] position of a full slot in the lower storage, -1 for upper
  int* l_row_ptr = nullptr;  // [n+1]
  int* l_col = nullptr;      // [nl]
  int* u_row_ptr = nullptr;  // [n+1] mirror index: row i, j > i
  int* u_pos = nullptr;      // [nu] lower-storage position of (j, i)
  int* u_col = nullptr;      // [nu] j
};

// Per-Newton-iteration contact/friction BSR built by sorting (row,col) keys.
struct ContactWork {
  DevBuf<unsigned long long> keys, keys_alt;
  DevBuf<int> codes, codes_alt, flag, scan, start, nvalid;
  DevBuf<unsigned char> tmp;
  DevBuf<int> row_ptr, col;
  DevBuf<double> val;
  int nslots = 0;
  int nrows = 0;  // non-empty contact rows (= contact diagonal slots)
};

void gather_static(cudaStream_t st, const StaticPattern& sp, const double* stage, const double* mass,
                   double inv_h2, const uint8_t* fixed, double* val, double* lval, float* lval32 = nullptr);
int build_contact_pattern(cudaStream_t st, ContactWork& w, int ns, const int* nodes, const uint8_t* fixed, int n,
                          const double* stage);
void node_finalize(cudaStream_t st, int n, const double* x, const double* y, const double* mass, double inv_h2,
                   const uint8_t* fixed, const StaticPattern& sp, const double* grad_e, const double* lbar_e,
                   const double* sval, const ContactWork* cw, const double* grad_c, const double* lbar_c,
                   double* grad, double* e_node, int* group, double* dinv);

}  // namespace bal
