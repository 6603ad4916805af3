// geometry.cuh -- primitive-pair distance resolution (device), mirroring the readings of
// SURVEY Q2 (Euclidean distance), Q27 (type resolution, ties) and DESIGN.md R-EE1.
//   PT interior iff projected barycentrics u,v >= 0 and u+v <= 1; else min over 3 point-segments.
//   EE interior iff ||ea x eb||^2 > 1e-10 ||ea||^2 ||eb||^2 and s,t in [0,1]; else min over 4
//   point-segments.  point-segment: t<0 -> PP(p,a); t>1 -> PP(p,b); else PE.
//   Ties: higher-dimensional feature first, then lowest candidate index.
#pragma once
#include "common.cuh"

namespace bal {

enum : int { T_PP = 0, T_PE = 1, T_PT = 2, T_EE = 3 };

BAL_HD int type_nodes(int t) { return t == T_PP ? 2 : (t == T_PE ? 3 : 4); }

struct Resolved {
  int type;    // sub-type
  int loc[4];  // role-ordered local indices into the 4 input slots (-1 padded)
  double D;    // squared distance
};

BAL_D void point_segment(d3 p, d3 a, d3 b, double& D, int& typ, int& end) {
  const d3 e = b - a;
  const double ee = dot(e, e);
  const double t = dot(p - a, e) / ee;
  if (t < 0.0) {
    D = dot(p - a, p - a);
    typ = T_PP;
    end = 0;
  } else if (t > 1.0) {
    D = dot(p - b, p - b);
    typ = T_PP;
    end = 1;
  } else {
    const d3 c = cross(a - p, b - p);
    D = dot(c, c) / ee;
    typ = T_PE;
    end = 0;
  }
}

BAL_D void ps_locals(int pl, int al, int bl, int typ, int end, int loc[4]) {
  loc[0] = pl;
  loc[3] = -1;
  if (typ == T_PE) {
    loc[1] = al;
    loc[2] = bl;
  } else {
    loc[1] = end ? bl : al;
    loc[2] = -1;
  }
}

BAL_D void take_min(Resolved& best, bool& have, double D, int typ, const int loc[4]) {
  if (!have || D < best.D || (D == best.D && typ > best.type)) {
    best.D = D;
    best.type = typ;
    for (int i = 0; i < 4; ++i) best.loc[i] = loc[i];
    have = true;
  }
}

BAL_D Resolved resolve_pt(d3 P, d3 A, d3 B, d3 C) {
  Resolved r;
  const d3 e1 = B - A, e2 = C - A, w = P - A;
  const double a11 = dot(e1, e1), a12 = dot(e1, e2), a22 = dot(e2, e2);
  const double r1 = dot(e1, w), r2 = dot(e2, w);
  const double det = a11 * a22 - a12 * a12;
  const double u = (a22 * r1 - a12 * r2) / det;
  const double v = (a11 * r2 - a12 * r1) / det;
  if (u >= 0.0 && v >= 0.0 && u + v <= 1.0) {
    const d3 n = cross(e1, e2);
    const double wn = dot(w, n);
    r.D = wn * wn / dot(n, n);
    r.type = T_PT;
    r.loc[0] = 0; r.loc[1] = 1; r.loc[2] = 2; r.loc[3] = 3;
    return r;
  }
  bool have = false;
  int loc[4];
  double D;
  int typ, end;
  point_segment(P, A, B, D, typ, end);
  ps_locals(0, 1, 2, typ, end, loc);
  take_min(r, have, D, typ, loc);
  point_segment(P, B, C, D, typ, end);
  ps_locals(0, 2, 3, typ, end, loc);
  take_min(r, have, D, typ, loc);
  point_segment(P, C, A, D, typ, end);
  ps_locals(0, 3, 1, typ, end, loc);
  take_min(r, have, D, typ, loc);
  return r;
}

BAL_D Resolved resolve_ee(d3 A0, d3 A1, d3 B0, d3 B1) {
  Resolved r;
  const d3 ea = A1 - A0, eb = B1 - B0, rr = A0 - B0;
  const double a = dot(ea, ea), b = dot(ea, eb), c = dot(eb, eb);
  const double d = dot(ea, rr), e = dot(eb, rr);
  const double den = a * c - b * b;
  if (den > 1e-10 * a * c) {
    const double s = (b * e - c * d) / den;
    const double t = (a * e - b * d) / den;
    if (s >= 0.0 && s <= 1.0 && t >= 0.0 && t <= 1.0) {
      const d3 n = cross(ea, eb);
      const double rn = dot(rr, n);
      r.D = rn * rn / dot(n, n);
      r.type = T_EE;
      r.loc[0] = 0; r.loc[1] = 1; r.loc[2] = 2; r.loc[3] = 3;
      return r;
    }
  }
  bool have = false;
  int loc[4];
  double D;
  int typ, end;
  point_segment(A0, B0, B1, D, typ, end);
  ps_locals(0, 2, 3, typ, end, loc);
  take_min(r, have, D, typ, loc);
  point_segment(A1, B0, B1, D, typ, end);
  ps_locals(1, 2, 3, typ, end, loc);
  take_min(r, have, D, typ, loc);
  point_segment(B0, A0, A1, D, typ, end);
  ps_locals(2, 0, 1, typ, end, loc);
  take_min(r, have, D, typ, loc);
  point_segment(B1, A0, A1, D, typ, end);
  ps_locals(3, 0, 1, typ, end, loc);
  take_min(r, have, D, typ, loc);
  return r;
}

// Resolve a feature pair of feature type ftype given its 4 role-ordered points.
BAL_D Resolved resolve(int ftype, d3 X0, d3 X1, d3 X2, d3 X3) {
  if (ftype == T_PT) return resolve_pt(X0, X1, X2, X3);
  if (ftype == T_EE) return resolve_ee(X0, X1, X2, X3);
  Resolved r;
  if (ftype == T_PE) {
    int typ, end;
    point_segment(X0, X1, X2, r.D, typ, end);
    r.type = typ;
    ps_locals(0, 1, 2, typ, end, r.loc);
    return r;
  }
  const d3 dd = X0 - X1;
  r.D = dot(dd, dd);
  r.type = T_PP;
  r.loc[0] = 0; r.loc[1] = 1; r.loc[2] = -1; r.loc[3] = -1;
  return r;
}

// Canonical constraint key from a resolved sub-type and role-ordered global ids (Q10/Q28):
// PP sorted; PE (p, sorted edge); PT (p, sorted tri); EE edges sorted, pair sorted.
struct Key {
  int t, n[4];
};
BAL_HD void sort2(int& a, int& b) {
  if (b < a) { int t = a; a = b; b = t; }
}
BAL_HD Key make_key(int typ, const int g[4]) {
  Key k;
  k.t = typ;
  k.n[0] = k.n[1] = k.n[2] = k.n[3] = -1;
  if (typ == T_PP) {
    int a = g[0], b = g[1];
    sort2(a, b);
    k.n[0] = a; k.n[1] = b;
  } else if (typ == T_PE) {
    int a = g[1], b = g[2];
    sort2(a, b);
    k.n[0] = g[0]; k.n[1] = a; k.n[2] = b;
  } else if (typ == T_PT) {
    int a = g[1], b = g[2], c = g[3];
    sort2(a, b); sort2(b, c); sort2(a, b);
    k.n[0] = g[0]; k.n[1] = a; k.n[2] = b; k.n[3] = c;
  } else {
    int a0 = g[0], a1 = g[1], b0 = g[2], b1 = g[3];
    sort2(a0, a1);
    sort2(b0, b1);
    if (b0 < a0 || (b0 == a0 && b1 < a1)) {
      int t0 = a0, t1 = a1;
      a0 = b0; a1 = b1; b0 = t0; b1 = t1;
    }
    k.n[0] = a0; k.n[1] = a1; k.n[2] = b0; k.n[3] = b1;
  }
  return k;
}

// 128-bit sortable key: hi = type<<62 | n0<<31 | n1 ; lo = n2<<31 | n3, with -1 -> 0x7fffffff.
BAL_HD unsigned long long key_hi(const Key& k) {
  auto f = [](int v) -> unsigned long long { return v < 0 ? 0x7fffffffull : (unsigned long long)v; };
  return ((unsigned long long)k.t << 62) | (f(k.n[0]) << 31) | f(k.n[1]);
}
BAL_HD unsigned long long key_lo(const Key& k) {
  auto f = [](int v) -> unsigned long long { return v < 0 ? 0x7fffffffull : (unsigned long long)v; };
  return (f(k.n[2]) << 31) | f(k.n[3]);
}
BAL_HD Key key_from(unsigned long long hi, unsigned long long lo) {
  auto g = [](unsigned long long v) -> int { return v == 0x7fffffffull ? -1 : (int)v; };
  Key k;
  k.t = (int)(hi >> 62);
  k.n[0] = g((hi >> 31) & 0x7fffffffull);
  k.n[1] = g(hi & 0x7fffffffull);
  k.n[2] = g((lo >> 31) & 0x7fffffffull);
  k.n[3] = g(lo & 0x7fffffffull);
  return k;
}

// barrier b(d; D) = -(d - D)^2 ln(d/D) for 0 < d < D, else 0
BAL_HD double barrier_b(double d, double Dh) {
  if (d >= Dh) return 0.0;
  const double t = d - Dh;
  return -t * t * log(d / Dh);
}
BAL_HD double barrier_b1(double d, double Dh) {
  if (d >= Dh) return 0.0;
  const double t = d - Dh;
  return -2.0 * t * log(d / Dh) - t * t / d;
}
BAL_HD double barrier_b2(double d, double Dh) {
  if (d >= Dh) return 0.0;
  const double t = d - Dh;
  return -2.0 * log(d / Dh) - 4.0 * t / d + t * t / (d * d);
}

}  // namespace bal
