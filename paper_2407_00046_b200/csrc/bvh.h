// bvh.h -- linear BVH (k_bvh.cu) and the collision-stage entry points (k_collision.cu).
#pragma once
#include "assemble.h"
#include "keys.h"

namespace bal {

struct Lbvh {
  int n = 0;
  DevBuf<double> lo, hi, nlo, nhi, part;
  DevBuf<unsigned long long> keys, keys2;
  DevBuf<int> left, right, parent, leaf_prim;
  DevBuf<unsigned> visits;
  DevBuf<unsigned char> tmp;
  // kind: nodes per primitive (2 edges, 3 triangles); boxes over the motion xa -> xb inflated by h
  void build(cudaStream_t st, int n, int kind, const int* prims, const double* xa, const double* xb, double h);
};

// mode 0: surface vertices vs triangle tree (PT pairs), mode 1: edges vs edge tree (EE pairs)
int query_pairs(cudaStream_t st, Lbvh& tree, int mode, int nq, const int* qprims, const int* tprims,
                const double* xa, const double* xb, double h, const uint8_t* fixed, DevBuf<int4>& out,
                DevBuf<int>& cnt);

// Candidate feature pairs (role-ordered) for one broad-phase query.
struct Candidates {
  DevBuf<int4> pt, ee;
  DevBuf<int> cnt;
  int npt = 0, nee = 0;
};

// Constraint set (unique resolved keys with d < dhat) at a position among candidates.
struct ConstraintSet {
  KeySorter ks;
  DevBuf<int> keys;          // [n][5] sorted
  DevBuf<double> d;          // [n] distance recomputed from the key
  DevBuf<unsigned long long> hi, lo;  // sorted packed keys
  DevBuf<int> cnt;
  int n = 0;
};

struct CollisionWork {
  Lbvh tri_tree, edge_tree;
  DevBuf<double> vals, part, scal;
  DevBuf<double> toi;
};

void broad_phase(cudaStream_t st, CollisionWork& w, Candidates& c, int V, const int* sverts, int F, const int* tris,
                 int E, const int* edges, const double* xa, const double* xb, double inflate, const uint8_t* fixed);
// returns |C(x)|; fills cs (keys, d sorted) and writes sigma * sum b(d) into *energy_dev, min d into *dmin_dev
int constraint_set(cudaStream_t st, ConstraintSet& cs, const Candidates& c, const double* x, double dhat);
void barrier_energy(cudaStream_t st, CollisionWork& w, const ConstraintSet& cs, double sigma, double dhat,
                    double* out_sum, double* out_min);
double ccd_step_toi(cudaStream_t st, CollisionWork& w, const Candidates& c, const double* x, const double* dx,
                    double dhat,
                    double d0frac);
void key_distances(cudaStream_t st, int n, const int* keys, const double* x, double* d);
void phi_al_energy(cudaStream_t st, CollisionWork& w, int n, const double* d, const double* mu, const double* s,
                   double sigma, double dhat, double* out_sum, double* out_min, double* out_abs_sum);

}  // namespace bal
