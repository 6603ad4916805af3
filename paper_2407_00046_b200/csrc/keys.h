// keys.h -- 128-bit constraint-key sort / unique helpers and the stencil set (A u A').
#pragma once
#include "assemble.h"

namespace bal {

// Sorts n packed (hi, lo) keys lexicographically (two stable 64-bit radix passes), carrying the
// original positions in idx; unique() then marks the first entry of every run of equal keys.
struct KeySorter {
  DevBuf<unsigned long long> hi, lo, lo_orig, hi2, lo2;
  DevBuf<int> idx, idx2, flag, scan, start, cnt;
  DevBuf<unsigned char> tmp;
  int idx_base = 0;
  int nuniq = 0;
  void prepare(int n);
  void sort(cudaStream_t st, int n);
  void sort_packed(cudaStream_t st, int n);  // hi/lo/idx filled by the caller
  int unique(cudaStream_t st, int n);        // fills start[0..nuniq] (start[nuniq] = n)
};

// Contact stencil set: union of A (resolved at x) and A' keys with flags / multipliers (Q22).
struct StencilSet {
  DevBuf<int> keys;  // [n][5]
  DevBuf<double> inA, inAp, mu, s;
  int n = 0;
  void reserve(int m) {
    keys.reserve(5 * (size_t)std::max(m, 1));
    inA.reserve(m);
    inAp.reserve(m);
    mu.reserve(m);
    s.reserve(m);
  }
};

void gather_u64(cudaStream_t st, int n, const unsigned long long* src, const int* idx, int base,
                unsigned long long* dst);
int stencil_union(cudaStream_t st, KeySorter& ks, int nA, const int* keysA, int nAp, const int* keysAp,
                  const double* ap_mu, const double* ap_s, StencilSet& out);

}  // namespace bal
