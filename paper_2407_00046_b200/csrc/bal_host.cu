// bal_host.cu -- C ABI (include/bal.h): context creation (mesh precompute, static BSR pattern,
// slot lists), assembly driver, SpMV and PCG drivers, test hooks.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <numeric>

#include "ctx.h"
#include "reduce.cuh"

using namespace bal;

void TsDev::build(int N, const std::vector<int>& lrow, const std::vector<int>& lcol, int val_bytes, cudaStream_t st) {
  ready = false;
  if (getenv("BAL_SPMV_GENERIC") != nullptr || N <= 0) return;
  int dev = 0, smem_max = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int env = getenv("BAL_TS_BUDGET") ? atoi(getenv("BAL_TS_BUDGET")) : 0;
  // largest block budget per tile whose kTsStages-stage ring fits the opt-in shared memory
  TsHost H;
  bool ok = false;
  // (kTsMinBlocks CTAs of it per SM; the driver reserves 1 KB of shared memory per CTA)
  int smem_sm = 0;
  CK(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  const size_t per_cta = std::min<size_t>((size_t)smem_max, (size_t)smem_sm / kTsMinBlocks) - 1024;
  for (int budget : {env > 0 ? env : 768, 704, 640, 576, 512, 448, 384, 320, 288, 256, 224, 192, 160, 128, 96, 64}) {
    if (!ts_build(N, lrow, lcol, budget, val_bytes, H)) return;
    if (H.smem <= per_cta) {
      ok = true;
      break;
    }
  }
  if (!ok) return;
  std::vector<int4> hd(H.ntiles + 1);
  for (int t = 0; t <= H.ntiles; ++t) {
    if (H.meta_off[t] / 16 >= (1ll << 31)) return;
    hd[t] = make_int4((int)(H.meta_off[t] / 16), H.tile_s0[t], H.tile_r0[t], 0);
  }
  desc.upload(hd.data(), hd.size(), st);
  pin_ptr.upload(H.pin_ptr.data(), H.pin_ptr.size(), st);
  meta.upload(H.meta.data(), std::max<size_t>(H.meta.size(), 16), st);
  part.reserve(3 * (size_t)std::max(H.nslots, 1));
  plan = TsPlan();
  plan.n = N;
  plan.ntiles = H.ntiles;
  plan.nslots = H.nslots;
  plan.desc = desc.ptr;
  plan.cap_rows = H.cap_rows;
  plan.o_crp = H.o_crp;
  plan.meta = meta.ptr;
  plan.pin_ptr = pin_ptr.ptr;
  plan.part = part.ptr;
  plan.o_meta = H.o_meta;
  plan.o_val = H.o_val;
  plan.o_vt = H.o_vt;
  plan.o_xv = H.o_xv;
  plan.stage_bytes = H.stage_bytes;
  plan.o_scratch = H.o_scratch;
  plan.cap_nb = H.cap_nb;
  plan.val_bytes = H.val_bytes;
  plan.cap_cs = H.cap_cs;
  plan.cap_tp = H.cap_tp;
  plan.smem = H.smem;
  plan.meta_bytes = (long long)H.meta.size();
  plan.ncross_total = H.ncross_total;
  CK(cudaStreamSynchronize(st));
  const int grid = ts_prepare(plan);
  ready = grid > 0;
  if (getenv("BAL_VERBOSE"))
    fprintf(stderr,
            "[bal-ts] N=%d tiles=%d grid=%d cap_nb=%d cap_rows=%d cap_x=%d cap_meta=%d smem=%zu slots=%d "
            "cross=%lld meta=%lld B\n",
            N, H.ntiles, grid, H.cap_nb, H.cap_rows, H.cap_x, H.cap_meta, H.smem, H.nslots, H.ncross_total,
            (long long)H.meta.size());
}

bal::Bsr bal_ctx::static_bsr() const {
  Bsr b;
  b.n = N;
  if (loaded_bsr) {
    b.nnzb = lb_nl;
    b.row_ptr = lb_lrow.ptr;
    b.col = lb_lcol.ptr;
    b.val = lb_lval.ptr;
    b.val32 = lb_lval32.ptr;
    b.m_row_ptr = lb_urow.ptr;
    b.m_pos = lb_upos.ptr;
    b.m_col = lb_ucol.ptr;
    b.nmirror = lb_nu;
    lb_ts.wire(b);
  } else if (sp_sym) {
    b.nnzb = sp.nl;
    b.row_ptr = sp.l_row_ptr;
    b.col = sp.l_col;
    b.val = lval.ptr;
    b.val32 = lval32.ptr;
    b.m_row_ptr = sp.u_row_ptr;
    b.m_pos = sp.u_pos;
    b.m_col = sp.u_col;
    b.nmirror = sp.nu;
    sp_ts.wire(b);
  } else {
    b.nnzb = sp.nnzb;
    b.row_ptr = sp.row_ptr;
    b.col = sp.col;
    b.val = sval.ptr;
    if (spmv_mode() == 2) b.tile_cap_s = sp.tile_cap_full;
  }
  return b;
}
bal::Bsr bal_ctx::contact_bsr() const {
  Bsr b;
  b.n = N;
  if (loaded_bsr || cw.nslots == 0) return b;
  b.nnzb = cw.nslots;
  b.row_ptr = cw.row_ptr.ptr;
  b.col = cw.col.ptr;
  b.val = cw.val.ptr;
  return b;
}

namespace {

struct MeshError : std::runtime_error {
  explicit MeshError(const std::string& s) : std::runtime_error(s) {}
};
struct ArgError : std::runtime_error {
  explicit ArgError(const std::string& s) : std::runtime_error(s) {}
};

template <typename F>
bal_status guard(bal_ctx* c, F&& f) {
  try {
    if (c) CK(cudaSetDevice(c->device));
    return f();
  } catch (const OomError& e) {
    if (c) c->err = e.what();
    return BAL_E_OOM;
  } catch (const CudaError& e) {
    if (c) c->err = e.what();
    return BAL_E_CUDA;
  } catch (const MeshError& e) {
    if (c) c->err = e.what();
    return BAL_E_BAD_MESH;
  } catch (const ArgError& e) {
    if (c) c->err = e.what();
    return BAL_E_INVALID_ARG;
  } catch (const std::invalid_argument& e) {
    if (c) c->err = e.what();
    return BAL_E_INVALID_ARG;
  } catch (const NcclError& e) {
    if (c) c->err = e.what();
    return BAL_E_NCCL;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return BAL_E_CUDA;
  }
}

// ------------------------------------------------------------------ mesh precomputation
void precompute(bal_ctx* c, const bal_mesh* m, const bal_material* mats, int nmat) {
  const int N = m->n_nodes, T = m->n_tets;
  if (N <= 0 || T < 0 || !m->rest_x || (T > 0 && (!m->tets || !m->tet_material)) || !m->node_fixed)
    throw ArgError("bal_init: bad mesh arguments");
  c->N = N;
  c->T = T;
  const double* X = m->rest_x;
  std::vector<double> Dm_inv(9 * (size_t)T), vol(T), mu(T), lam(T), mass(N, 0.0);
  std::vector<unsigned char> tmodel(T, 0);
  std::vector<int4> tets(T);
  for (int e = 0; e < T; ++e) {
    int t[4];
    for (int a = 0; a < 4; ++a) {
      t[a] = m->tets[4 * (size_t)e + a];
      if (t[a] < 0 || t[a] >= N) throw MeshError("tet " + std::to_string(e) + " has an out-of-range node index");
    }
    tets[e] = make_int4(t[0], t[1], t[2], t[3]);
    const int mi = m->tet_material[e];
    if (mi < 0 || mi >= nmat) throw ArgError("tet " + std::to_string(e) + ": bad material index");
    double D[3][3];
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) D[r][k] = X[3 * (size_t)t[k + 1] + r] - X[3 * (size_t)t[0] + r];
    const double C00 = D[1][1] * D[2][2] - D[1][2] * D[2][1], C01 = D[1][2] * D[2][0] - D[1][0] * D[2][2],
                 C02 = D[1][0] * D[2][1] - D[1][1] * D[2][0];
    const double det = D[0][0] * C00 + D[0][1] * C01 + D[0][2] * C02;
    if (!(det > 0.0)) throw MeshError("inverted or degenerate rest tet " + std::to_string(e));
    double inv[3][3];
    inv[0][0] = C00 / det;
    inv[1][0] = C01 / det;
    inv[2][0] = C02 / det;
    inv[0][1] = (D[0][2] * D[2][1] - D[0][1] * D[2][2]) / det;
    inv[1][1] = (D[0][0] * D[2][2] - D[0][2] * D[2][0]) / det;
    inv[2][1] = (D[0][1] * D[2][0] - D[0][0] * D[2][1]) / det;
    inv[0][2] = (D[0][1] * D[1][2] - D[0][2] * D[1][1]) / det;
    inv[1][2] = (D[0][2] * D[1][0] - D[0][0] * D[1][2]) / det;
    inv[2][2] = (D[0][0] * D[1][1] - D[0][1] * D[1][0]) / det;
    for (int i = 0; i < 9; ++i) Dm_inv[9 * (size_t)e + i] = inv[i / 3][i % 3];
    vol[e] = det / 6.0;
    const double E = mats[mi].E, nu = mats[mi].nu, rho = mats[mi].rho;
    mu[e] = E / (2.0 * (1.0 + nu));
    lam[e] = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    if (mats[mi].model != BAL_MODEL_NEO_HOOKEAN && mats[mi].model != BAL_MODEL_ARAP)
      throw std::invalid_argument("bal_init: unknown material model");
    tmodel[e] = (unsigned char)mats[mi].model;
    for (int a = 0; a < 4; ++a) mass[t[a]] += rho * vol[e] / 4.0;
  }
  c->h_fixed.assign(m->node_fixed, m->node_fixed + N);
  c->h_mass = mass;
  double msum = 0.0;
  int nf = 0;
  for (int i = 0; i < N; ++i)
    if (!c->h_fixed[i]) {
      msum += mass[i];
      ++nf;
    }
  c->n_free = nf;
  c->mean_free_mass = nf ? msum / nf : 1.0;

  // ---- surface triangles: faces referenced once, oriented away from the opposite vertex
  struct Face {
    int k[3];
    int f[3];
    int opp;
  };
  std::vector<Face> faces;
  faces.reserve(4 * (size_t)T);
  static const int fl[4][4] = {{0, 1, 2, 3}, {0, 1, 3, 2}, {0, 2, 3, 1}, {1, 2, 3, 0}};
  for (int e = 0; e < T; ++e) {
    const int t[4] = {tets[e].x, tets[e].y, tets[e].z, tets[e].w};
    for (int q = 0; q < 4; ++q) {
      Face f;
      f.f[0] = t[fl[q][0]];
      f.f[1] = t[fl[q][1]];
      f.f[2] = t[fl[q][2]];
      f.opp = t[fl[q][3]];
      int k3[3] = {f.f[0], f.f[1], f.f[2]};
      std::sort(k3, k3 + 3);
      f.k[0] = k3[0];
      f.k[1] = k3[1];
      f.k[2] = k3[2];
      faces.push_back(f);
    }
  }
  std::sort(faces.begin(), faces.end(), [](const Face& a, const Face& b) {
    return std::lexicographical_compare(a.k, a.k + 3, b.k, b.k + 3);
  });
  std::vector<std::array<int, 3>> tris;
  for (size_t i = 0; i < faces.size();) {
    size_t j = i + 1;
    while (j < faces.size() && std::equal(faces[j].k, faces[j].k + 3, faces[i].k)) ++j;
    if (j - i == 1) {
      Face f = faces[i];
      const double* a = X + 3 * (size_t)f.f[0];
      const double* b = X + 3 * (size_t)f.f[1];
      const double* cc = X + 3 * (size_t)f.f[2];
      const double* o = X + 3 * (size_t)f.opp;
      const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, v[3] = {cc[0] - a[0], cc[1] - a[1], cc[2] - a[2]};
      const double n[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
      const double s = n[0] * (o[0] - a[0]) + n[1] * (o[1] - a[1]) + n[2] * (o[2] - a[2]);
      if (s > 0) std::swap(f.f[1], f.f[2]);
      tris.push_back({f.f[0], f.f[1], f.f[2]});
    }
    i = j;
  }
  for (int i = 0; i < m->n_obstacle_tris; ++i) {
    std::array<int, 3> t3;
    for (int a = 0; a < 3; ++a) {
      t3[a] = m->obstacle_tris[3 * (size_t)i + a];
      if (t3[a] < 0 || t3[a] >= N) throw MeshError("obstacle triangle index out of range");
      if (!c->h_fixed[t3[a]]) throw MeshError("obstacle triangle references a free node");
    }
    tris.push_back(t3);
  }
  std::vector<std::array<int, 2>> edges;
  edges.reserve(3 * tris.size());
  for (auto& t3 : tris)
    for (int a = 0; a < 3; ++a) {
      int u = t3[a], v = t3[(a + 1) % 3];
      if (v < u) std::swap(u, v);
      edges.push_back({u, v});
    }
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  std::vector<int> sv;
  sv.reserve(3 * tris.size());
  for (auto& t3 : tris)
    for (int a = 0; a < 3; ++a) sv.push_back(t3[a]);
  std::sort(sv.begin(), sv.end());
  sv.erase(std::unique(sv.begin(), sv.end()), sv.end());
  c->F = (int)tris.size();
  c->E = (int)edges.size();
  c->V = (int)sv.size();

  // ---- static BSR pattern over mesh adjacency (+ every diagonal)
  std::vector<int> n2t_ptr(N + 1, 0);
  for (int e = 0; e < T; ++e) {
    n2t_ptr[tets[e].x + 1]++;
    n2t_ptr[tets[e].y + 1]++;
    n2t_ptr[tets[e].z + 1]++;
    n2t_ptr[tets[e].w + 1]++;
  }
  for (int i = 0; i < N; ++i) n2t_ptr[i + 1] += n2t_ptr[i];
  std::vector<int> n2t(n2t_ptr[N]);
  {
    std::vector<int> fill(n2t_ptr.begin(), n2t_ptr.end() - 1);
    for (int e = 0; e < T; ++e) {
      n2t[fill[tets[e].x]++] = e;
      n2t[fill[tets[e].y]++] = e;
      n2t[fill[tets[e].z]++] = e;
      n2t[fill[tets[e].w]++] = e;
    }
  }
  std::vector<int> row_ptr(N + 1, 0), col;
  col.reserve((size_t)N * 12);
  std::vector<int> nb;
  for (int i = 0; i < N; ++i) {
    nb.clear();
    nb.push_back(i);
    for (int q = n2t_ptr[i]; q < n2t_ptr[i + 1]; ++q) {
      const int4 t = tets[n2t[q]];
      nb.push_back(t.x);
      nb.push_back(t.y);
      nb.push_back(t.z);
      nb.push_back(t.w);
    }
    std::sort(nb.begin(), nb.end());
    nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    col.insert(col.end(), nb.begin(), nb.end());
    row_ptr[i + 1] = (int)col.size();
  }
  const int nnzb = (int)col.size();
  std::vector<int> slot_row(nnzb), diag_pos(N);
  for (int i = 0; i < N; ++i)
    for (int s = row_ptr[i]; s < row_ptr[i + 1]; ++s) {
      slot_row[s] = i;
      if (col[s] == i) diag_pos[i] = s;
    }
  auto find_slot = [&](int i, int j) {
    auto b = col.begin() + row_ptr[i], e = col.begin() + row_ptr[i + 1];
    return (int)(std::lower_bound(b, e, j) - col.begin());
  };
  std::vector<int> slot_ptr(nnzb + 1, 0), slot_code(16 * (size_t)T);
  std::vector<int> tslot(16 * (size_t)T);
  for (int e = 0; e < T; ++e) {
    const int t[4] = {tets[e].x, tets[e].y, tets[e].z, tets[e].w};
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) {
        const int s = find_slot(t[a], t[b]);
        tslot[16 * (size_t)e + 4 * a + b] = s;
        slot_ptr[s + 1]++;
      }
  }
  for (int s = 0; s < nnzb; ++s) slot_ptr[s + 1] += slot_ptr[s];
  {
    std::vector<int> fill(slot_ptr.begin(), slot_ptr.end() - 1);
    for (int e = 0; e < T; ++e)
      for (int ab = 0; ab < 16; ++ab) slot_code[fill[tslot[16 * (size_t)e + ab]]++] = e * 16 + ab;
  }

  // ---- upload
  cudaStream_t st = c->st;
  c->tets.upload(tets.data(), T, st);
  c->Dm_inv.upload(Dm_inv.data(), Dm_inv.size(), st);
  c->vol.upload(vol.data(), T, st);
  c->mu.upload(mu.data(), T, st);
  c->any_arap = std::find(tmodel.begin(), tmodel.end(), (unsigned char)BAL_MODEL_ARAP) != tmodel.end();
  if (c->any_arap) c->tmodel.upload(tmodel.data(), T, st);
  c->lam.upload(lam.data(), T, st);
  c->mass.upload(mass.data(), N, st);
  c->fixed.upload(c->h_fixed.data(), N, st);
  std::vector<int> trisf(3 * tris.size()), edgesf(2 * edges.size());
  for (size_t i = 0; i < tris.size(); ++i)
    for (int a = 0; a < 3; ++a) trisf[3 * i + a] = tris[i][a];
  for (size_t i = 0; i < edges.size(); ++i) {
    edgesf[2 * i] = edges[i][0];
    edgesf[2 * i + 1] = edges[i][1];
  }
  c->tris.upload(trisf.data(), trisf.size(), st);
  c->edges.upload(edgesf.data(), edgesf.size(), st);
  c->sverts.upload(sv.data(), sv.size(), st);
  c->dist.adj_ptr = row_ptr;  // host copy of the static pattern for the halo plan (kept if distributed)
  c->dist.adj_col = col;
  c->sp_row_ptr.upload(row_ptr.data(), row_ptr.size(), st);
  c->sp_col.upload(col.data(), col.size(), st);
  c->sp_slot_row.upload(slot_row.data(), slot_row.size(), st);
  c->sp_diag_pos.upload(diag_pos.data(), diag_pos.size(), st);
  c->sp_slot_ptr.upload(slot_ptr.data(), slot_ptr.size(), st);
  c->sp_slot_code.upload(slot_code.data(), slot_code.size(), st);
  c->sp.n = N;
  c->sp.nnzb = nnzb;
  c->sp.row_ptr = c->sp_row_ptr.ptr;
  c->sp.col = c->sp_col.ptr;
  c->sp.slot_row = c->sp_slot_row.ptr;
  c->sp.diag_pos = c->sp_diag_pos.ptr;
  c->sp.slot_ptr = c->sp_slot_ptr.ptr;
  c->sp.slot_code = c->sp_slot_code.ptr;
  // symmetric copy for the SpMV: lower + diagonal slots in row order, and per row i the mirror
  // index of its upper slots (j > i) -> lower-storage position of (j, i)
  {
    std::vector<int> lpos(nnzb, -1), lrow(N + 1, 0), lcol, urow(N + 1, 0), upos, ucol;
    lcol.reserve((nnzb + N) / 2);
    for (int i = 0; i < N; ++i) {
      for (int s2 = row_ptr[i]; s2 < row_ptr[i + 1]; ++s2)
        if (col[s2] <= i) {
          lpos[s2] = (int)lcol.size();
          lcol.push_back(col[s2]);
        }
      lrow[i + 1] = (int)lcol.size();
    }
    for (int i = 0; i < N; ++i) {
      for (int s2 = row_ptr[i]; s2 < row_ptr[i + 1]; ++s2)
        if (col[s2] > i) {
          const int j = col[s2];
          upos.push_back(lpos[find_slot(j, i)]);
          ucol.push_back(j);
        }
      urow[i + 1] = (int)ucol.size();
    }
    c->sp.nl = (int)lcol.size();
    c->sp.nu = (int)ucol.size();
    c->sp_lpos.upload(lpos.data(), lpos.size(), st);
    c->sp_lrow.upload(lrow.data(), lrow.size(), st);
    lcol.resize(lcol.size() + 8, 0);  // 16-byte slack: the tile bulk copies round the range up
    c->sp_lcol.upload(lcol.data(), lcol.size(), st);
    lcol.resize(lcol.size() - 8);
    c->sp_urow.upload(urow.data(), urow.size(), st);
    c->sp_upos.upload(upos.data(), std::max<size_t>(upos.size(), 1), st);
    c->sp_ucol.upload(ucol.data(), std::max<size_t>(ucol.size(), 1), st);
    c->sp.lpos = c->sp_lpos.ptr;
    c->sp.l_row_ptr = c->sp_lrow.ptr;
    c->sp.l_col = c->sp_lcol.ptr;
    c->sp.u_row_ptr = c->sp_urow.ptr;
    c->sp.u_pos = c->sp_upos.ptr;
    c->sp.u_col = c->sp_ucol.ptr;
    c->sp_sym = spmv_symmetric_enabled();
    if (c->sp_sym) {
      c->lval.reserve(9 * (size_t)std::max(c->sp.nl, 1) + 2);  // + 16 B slack for the bulk copies
      if (c->prm.flags & BAL_FP32_MATRIX) c->lval32.reserve(9 * (size_t)std::max(c->sp.nl, 1) + 4);
      c->sp_ts.build(N, lrow, lcol, (c->prm.flags & BAL_FP32_MATRIX) ? 36 : 72, st);
    }
    for (int r0 = 0; r0 < N; r0 += kSpmvTileRows)
      c->sp.tile_cap_full = std::max(c->sp.tile_cap_full,
                                     row_ptr[std::min(N, r0 + kSpmvTileRows)] - row_ptr[r0]);
    spmv_init_grids();
    spmv_prepare(c->static_bsr());
  }
  c->sval.reserve(9 * (size_t)nnzb);
  c->stage_e.reserve(90 * (size_t)std::max(T, 1));
  c->grad_e.reserve(12 * (size_t)std::max(T, 1));
  c->lbar_e.reserve(std::max(T, 1));
  c->grad.reserve(3 * (size_t)N);
  c->e_node.reserve(N);
  c->dinv.reserve(6 * (size_t)N);
  c->group.reserve(N);
  c->grp_c.reserve(N);
  c->y.reserve(3 * (size_t)N);
  c->xt.reserve(3 * (size_t)N);
  for (auto* b : {&c->pr, &c->pz, &c->pp, &c->pq, &c->px, &c->ps, &c->tmp_a, &c->tmp_b}) b->reserve(3 * (size_t)N);
  c->upart.reserve(3 * (size_t)kVecBlocks);  // (r,u), (r,r) pairs + (x,x) for App. B criterion (ii)
  c->dpart.reserve(4 * (size_t)kSMs);
  c->partials.reserve((size_t)kRedBlocks * kMaxGroups * 4 + 16 * kSMs * 4);
  c->red.reserve(kRedBlocks + 16);  // [0, kRedBlocks) partials, then scalar outputs
  c->counter.reserve(1);
  CK(cudaMemsetAsync(c->counter.ptr, 0, sizeof(unsigned), st));
  c->scal.reserve(1);
  c->gscal.reserve(1);
  c->hist.reserve(std::max(c->prm.max_pcg, 1) + 8);
  CK(cudaMallocHost(&c->h_scal, 3 * sizeof(PcgScal)));  // [0] current, [1..2] graph ping-pong copies
  CK(cudaStreamSynchronize(st));
}

}  // namespace

// ================================================================== assembly driver
namespace bal {

// Assemble at x with the current contact/friction stencil sets (c->cset, c->fr_*) and predictor y.
void run_assembly(bal_ctx* c, const double* x, const double* y, double sigma) {
  cudaStream_t st = c->st;
  const int T = c->T, N = c->N;
  launch_elastic(st, T, x, c->tets.ptr, c->Dm_inv.ptr, c->vol.ptr, c->mu.ptr, c->lam.ptr, c->any_arap ? c->tmodel.ptr : nullptr,
                 c->stage_e.ptr,
                 c->grad_e.ptr, c->lbar_e.ptr);
  const int nc = c->cset.n, nf = c->n_fric, ns = nc + nf;
  c->n_contact = nc;
  if (ns > 0) {
    c->stage_c.reserve(90 * (size_t)ns);
    c->grad_c.reserve(12 * (size_t)ns);
    c->lbar_c.reserve(ns);
    c->nodes_c.reserve(4 * (size_t)ns);
    c->dist_c.reserve(ns);
    c->dphi_c.reserve(ns);
    launch_contact(st, nc, x, c->cset.keys.ptr, c->cset.inA.ptr, c->cset.inAp.ptr, c->cset.mu.ptr, c->cset.s.ptr,
                   sigma, c->prm.dhat, c->stage_c.ptr, c->grad_c.ptr, c->lbar_c.ptr, c->nodes_c.ptr,
                   c->dist_c.ptr, c->dphi_c.ptr);
    if (nf > 0)
      launch_friction(st, nf, x, c->xt.ptr, c->fr_keys.ptr, c->fr_gam.ptr, c->fr_nrm.ptr, c->fr_lam.ptr,
                      c->prm.chi, c->prm.eps_v * c->prm.h, c->stage_c.ptr + 90 * (size_t)nc,
                      c->grad_c.ptr + 12 * (size_t)nc, c->lbar_c.ptr + nc, c->nodes_c.ptr + 4 * (size_t)nc);
  }
  const double inv_h2 = 1.0 / (c->prm.h * c->prm.h);
  gather_static(st, c->sp, c->stage_e.ptr, c->mass.ptr, inv_h2, c->fixed.ptr, c->sval.ptr,
                c->sp_sym ? c->lval.ptr : nullptr, c->sp_sym ? c->lval32.ptr : nullptr);
  build_contact_pattern(st, c->cw, ns, c->nodes_c.ptr, c->fixed.ptr, N, c->stage_c.ptr);
  if (ns == 0) c->cw.nslots = 0;
  node_finalize(st, N, x, y, c->mass.ptr, inv_h2, c->fixed.ptr, c->sp, c->grad_e.ptr, c->lbar_e.ptr, c->sval.ptr,
                &c->cw, c->grad_c.ptr, c->lbar_c.ptr, c->grad.ptr, c->e_node.ptr, c->group.ptr, c->dinv.ptr);
  c->launches += 6;
  c->loaded_bsr = false;
}

}  // namespace bal

// ================================================================== C ABI
static thread_local std::string g_init_err;

static void fill_view(const bal_ctx* c, bal_system_view* v) {
  std::memset(v, 0, sizeof(*v));
  v->n_nodes = c->N;
  v->nnzb_static = c->sp.nnzb;
  v->static_row_ptr = c->sp.row_ptr;
  v->static_col = c->sp.col;
  v->static_val = c->sval.ptr;
  v->nnzb_contact = c->cw.nslots;
  v->contact_row_ptr = c->cw.nslots ? c->cw.row_ptr.ptr : nullptr;
  v->contact_col = c->cw.nslots ? c->cw.col.ptr : nullptr;
  v->contact_val = c->cw.nslots ? c->cw.val.ptr : nullptr;
  v->diag_inv = c->dinv.ptr;
  v->grad = c->grad.ptr;
  v->e_node = c->e_node.ptr;
  v->group = c->group.ptr;
  v->n_elastic = c->T;
  v->elastic_blocks = c->stage_e.ptr;
  v->elastic_lbar = c->lbar_e.ptr;
  v->n_contact_stencils = c->n_contact + c->n_fric;
  v->contact_blocks = c->stage_c.ptr;
  v->contact_lbar = c->lbar_c.ptr;
  v->contact_stencil_nodes = c->nodes_c.ptr;
  v->n_friction_stencils = c->n_fric;
  v->contact_grad = c->grad_c.ptr;
}

extern "C" {

bal_status bal_init(const bal_mesh* mesh, const bal_material* materials, int32_t n_materials,
                    const bal_params* params, const bal_dist* dist, bal_ctx** out) {
  if (!out) return BAL_E_INVALID_ARG;
  *out = nullptr;
  if (!mesh || !materials || n_materials <= 0 || !params) return BAL_E_INVALID_ARG;
  if (dist && (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world ||
               ((dist->host_allreduce == nullptr) != (dist->host_exchange == nullptr))))
    return BAL_E_INVALID_ARG;
  const int device = dist ? dist->device : 0;
  bal_ctx* c = new bal_ctx();
  c->device = device;
  c->prm = *params;
  const bal_status s = guard(c, [&]() {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ArgError("bal_init: no such CUDA device");
    CK(cudaSetDevice(device));
    // blocking stream: implicitly ordered after work on the legacy default stream (e.g. a torch
    // H2D copy of x_t issued just before bal_step), so callers need no explicit sync
    CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamDefault));
    c->st = c->own_stream;
    if (!(c->prm.h > 0) || !(c->prm.dhat > 0)) throw ArgError("bal_init: h and dhat must be > 0");
    precompute(c, mesh, materials, n_materials);
    if (dist) dist_init(c, dist);
    if (!c->dist.active) {
      c->dist.adj_ptr.clear();
      c->dist.adj_ptr.shrink_to_fit();
      c->dist.adj_col.clear();
      c->dist.adj_col.shrink_to_fit();
    }
    return BAL_OK;
  });
  if (s != BAL_OK) {
    g_init_err = c->err;  // reachable through bal_last_error(NULL)
    bal_destroy(c);
    return s;
  }
  *out = c;
  return BAL_OK;
}

bal_status bal_set_stream(bal_ctx* c, void* stream) {
  if (!c) return BAL_E_INVALID_ARG;
  c->st = stream ? (cudaStream_t)stream : c->own_stream;
  return BAL_OK;
}

bal_status bal_assemble(bal_ctx* c, const double* x, const bal_contact_state* cs, bal_system_view* v) {
  if (!c || !x || !cs) return BAL_E_INVALID_ARG;
  return guard(c, [&]() {
    cudaStream_t st = c->st;
    const int N = c->N;
    if (cs->y) c->y.upload(cs->y, 3 * (size_t)N, st);
    else CK(cudaMemcpyAsync(c->y.ptr, x, 3 * (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (cs->x_t) c->xt.upload(cs->x_t, 3 * (size_t)N, st);
    // contact stencil set = A u A'
    DevBuf<int> dA, dAp;
    DevBuf<double> dmu, ds;
    if (cs->n_active) dA.upload(cs->active_keys, 5 * (size_t)cs->n_active, st);
    if (cs->n_aprime) {
      dAp.upload(cs->aprime_keys, 5 * (size_t)cs->n_aprime, st);
      dmu.upload(cs->aprime_mu, cs->n_aprime, st);
      ds.upload(cs->aprime_s, cs->n_aprime, st);
    }
    stencil_union(st, c->ks, cs->n_active, dA.ptr, cs->n_aprime, dAp.ptr, dmu.ptr, ds.ptr, c->cset);
    c->n_fric = cs->n_friction;
    if (cs->n_friction) {
      c->fr_keys.upload(cs->friction_keys, 5 * (size_t)cs->n_friction, st);
      c->fr_gam.upload(cs->friction_gamma, 4 * (size_t)cs->n_friction, st);
      c->fr_nrm.upload(cs->friction_n, 3 * (size_t)cs->n_friction, st);
      c->fr_lam.upload(cs->friction_lambda, cs->n_friction, st);
      if (!cs->x_t) throw ArgError("bal_assemble: friction needs x_t");
    }
    run_assembly(c, x, c->y.ptr, cs->sigma);
    CK(cudaStreamSynchronize(st));
    if (v) fill_view(c, v);
    return BAL_OK;
  });
}

bal_status bal_get_system(bal_ctx* c, bal_system_view* v) {
  if (!c || !v) return BAL_E_INVALID_ARG;
  return guard(c, [&]() {
    CK(cudaStreamSynchronize(c->st));
    fill_view(c, v);
    return BAL_OK;
  });
}

bal_status bal_spmv(bal_ctx* c, const double* v, double* y) {
  if (!c || !v || !y) return BAL_E_INVALID_ARG;
  return guard(c, [&]() {
    launch_spmv(c->st, c->static_bsr(), c->contact_bsr(), v, y);
    c->launches += ts_usable(c->static_bsr()) ? 2 : 1;
    CK(cudaStreamSynchronize(c->st));
    return BAL_OK;
  });
}

bal_status bal_spmv_rows(bal_ctx* c, int32_t r0, int32_t r1, const double* v, double* y) {
  if (!c || !v || !y || r0 < 0 || r1 < r0 || r1 > c->N) return BAL_E_INVALID_ARG;
  if (r0 % kPartAlign != 0 || (r1 != c->N && r1 % kPartAlign != 0)) return BAL_E_INVALID_ARG;
  return guard(c, [&]() {
    Bsr S = c->static_bsr();
    S.r0 = r0;
    S.r1 = r1;
    S.ts = nullptr;  // the partitioned path's row-range kernel (pcg_dist.cu)
    if (r1 > r0) launch_spmv(c->st, S, c->contact_bsr(), v, y);
    c->launches += 1;
    CK(cudaStreamSynchronize(c->st));
    return BAL_OK;
  });
}

bal_status bal_pcg(bal_ctx* c, const double* rhs, const double* x0, double* x_out, const bal_pcg_opts* o,
                   bal_pcg_stats* stats) {
  if (!c || !rhs || !x_out) return BAL_E_INVALID_ARG;
  return guard(c, [&]() {
    bal_pcg_opts d{};
    d.warm_start = (c->prm.flags & BAL_NO_WARMSTART) ? 0 : 1;
    d.rel_tol = c->prm.pcg_rel_tol;
    d.stall_window = c->prm.pcg_stall_window;
    d.max_iters = c->prm.max_pcg;
    d.ws_rel_tol = c->prm.ws_rel_tol;
    d.ws_max_iters = c->prm.ws_max_iters;
    const bal_pcg_opts& op = o ? *o : d;
    if (op.max_iters + 8 > (int)c->hist.cap) c->hist.reserve(op.max_iters + 8);
    pcg_solve(c, rhs, x0, x_out, op.warm_start != 0 && x0 == nullptr, op.rel_tol, op.stall_window, op.max_iters,
              op.ws_rel_tol, op.ws_max_iters, stats);
    CK(cudaStreamSynchronize(c->st));
    return BAL_OK;
  });
}

bal_status bal_load_bsr(bal_ctx* c, const bal_bsr_host* b) {
  if (!c || !b || b->n_nodes != c->N) return BAL_E_INVALID_ARG;
  return guard(c, [&]() {
    cudaStream_t st = c->st;
    c->lb_row_ptr.upload(b->row_ptr, c->N + 1, st);
    c->lb_col.upload(b->col, b->nnzb, st);
    c->lb_val.upload(b->val, 9 * (size_t)b->nnzb, st);
    c->lb_nnzb = b->nnzb;
    c->loaded_bsr = true;
    {  // symmetric copy (the SpMV reads the lower triangle; the loaded matrix must be symmetric)
      const int N = c->N;
      auto find = [&](int i, int j) {
        for (int s2 = b->row_ptr[i]; s2 < b->row_ptr[i + 1]; ++s2)
          if (b->col[s2] == j) return s2;
        throw ArgError("bal_load_bsr: pattern is not structurally symmetric");
      };
      std::vector<int> lpos(b->nnzb, -1), lrow(N + 1, 0), lcol, urow(N + 1, 0), upos, ucol;
      std::vector<double> lv;
      for (int i = 0; i < N; ++i) {
        for (int s2 = b->row_ptr[i]; s2 < b->row_ptr[i + 1]; ++s2)
          if (b->col[s2] <= i) {
            lpos[s2] = (int)lcol.size();
            lcol.push_back(b->col[s2]);
            lv.insert(lv.end(), b->val + 9 * (size_t)s2, b->val + 9 * (size_t)s2 + 9);
          }
        lrow[i + 1] = (int)lcol.size();
      }
      for (int i = 0; i < N; ++i) {
        for (int s2 = b->row_ptr[i]; s2 < b->row_ptr[i + 1]; ++s2)
          if (b->col[s2] > i) {
            upos.push_back(lpos[find(b->col[s2], i)]);
            ucol.push_back(b->col[s2]);
          }
        urow[i + 1] = (int)ucol.size();
      }
      c->lb_nl = (int)lcol.size();
      c->lb_nu = (int)ucol.size();
      lcol.resize(lcol.size() + 8, 0);
      lv.resize(lv.size() + 2, 0.0);
      c->lb_lrow.upload(lrow.data(), lrow.size(), st);
      c->lb_lcol.upload(lcol.data(), lcol.size(), st);
      c->lb_lval.upload(lv.data(), lv.size(), st);
      c->lb_urow.upload(urow.data(), urow.size(), st);
      c->lb_upos.upload(upos.data(), std::max<size_t>(upos.size(), 1), st);
      c->lb_ucol.upload(ucol.data(), std::max<size_t>(ucol.size(), 1), st);
      lcol.resize(lcol.size() - 8);
      if (c->prm.flags & BAL_FP32_MATRIX) {  // FP32 copy of the loaded blocks (rounded once)
        std::vector<float> lv32(lv.begin(), lv.end());
        lv32.resize(lv32.size() + 4, 0.f);
        c->lb_lval32.upload(lv32.data(), lv32.size(), st);
      }
      c->lb_ts.build(N, lrow, lcol, (c->prm.flags & BAL_FP32_MATRIX) ? 36 : 72, st);
    }

    // diagonal inverse from the loaded blocks (host: test path only)
    std::vector<double> dinv(6 * (size_t)c->N, 0.0);
    for (int i = 0; i < c->N; ++i) {
      double D[9] = {0};
      for (int s = b->row_ptr[i]; s < b->row_ptr[i + 1]; ++s)
        if (b->col[s] == i)
          for (int t = 0; t < 9; ++t) D[t] = b->val[9 * (size_t)s + t];
      const double a = D[0], bb = D[1], cc = D[2], d = D[4], f = D[5], k = D[8];
      const double A0 = d * k - f * f, A1 = cc * f - bb * k, A2 = bb * f - cc * d;
      const double det = a * A0 + bb * A1 + cc * A2;
      double* di = dinv.data() + 6 * (size_t)i;
      di[0] = A0 / det;
      di[1] = A1 / det;
      di[2] = A2 / det;
      di[3] = (a * k - cc * cc) / det;
      di[4] = (bb * cc - a * f) / det;
      di[5] = (a * d - bb * bb) / det;
    }
    c->dinv.upload(dinv.data(), dinv.size(), st);
    std::vector<int> g(c->N, 0);
    if (b->group) g.assign(b->group, b->group + c->N);
    for (int i = 0; i < c->N; ++i)
      if (c->h_fixed[i]) g[i] = INT32_MIN;
    c->group.upload(g.data(), g.size(), st);
    CK(cudaStreamSynchronize(st));
    return BAL_OK;
  });
}

bal_status bal_bench_spmv(bal_ctx* c, int32_t iters, double* mean_us) {
  if (!c || iters <= 0 || !mean_us) return BAL_E_INVALID_ARG;
  return guard(c, [&]() {
    cudaStream_t st = c->st;
    CK(cudaMemsetAsync(c->tmp_a.ptr, 0, 3 * (size_t)c->N * sizeof(double), st));
    launch_spmv(st, c->static_bsr(), c->contact_bsr(), c->tmp_a.ptr, c->tmp_b.ptr);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) launch_spmv(st, c->static_bsr(), c->contact_bsr(), c->tmp_a.ptr, c->tmp_b.ptr);
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    *mean_us = 1000.0 * ms / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c->launches += iters + 1;
    return BAL_OK;
  });
}

int64_t bal_kernel_launches(const bal_ctx* c) { return c ? c->launches : 0; }

int32_t bal_pcg_history(bal_ctx* c, double* out, int32_t max_n) {
  if (!c || !out || max_n <= 0) return BAL_E_INVALID_ARG;
  const int n = std::min(max_n, c->h_scal ? c->h_scal->k + 1 : 0);
  if (n <= 0) return 0;
  if (cudaMemcpy(out, c->hist.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return BAL_E_CUDA;
  return n;
}

int32_t bal_pcg_objective_history(bal_ctx* c, double* out, int32_t max_n) {
  if (!c || !out || max_n <= 0) return BAL_E_INVALID_ARG;
  const int n = std::min(max_n, c->h_scal ? c->h_scal->k + 1 : 0);
  if (n <= 0) return 0;
  if (cudaMemcpy(out, c->hist.ptr + c->h_scal->hcap, sizeof(double) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
    return BAL_E_CUDA;
  return n;
}

bal_status bal_spmv_counters(const bal_ctx* c, double* out) {
  if (!c || !out) return BAL_E_INVALID_ARG;
  out[0] = c->spmv_ms;
  out[1] = (double)c->spmv_count;
  out[2] = c->spmv_bytes_alg;
  out[3] = c->spmv_bytes_moved;
  return BAL_OK;
}

const char* bal_last_error(const bal_ctx* c) { return c ? c->err.c_str() : g_init_err.c_str(); }

void bal_destroy(bal_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  destroy_step_work(c);
  dist_destroy(c);
  if (c->ev_ready)
    for (cudaEvent_t e : c->ev)
      if (e) cudaEventDestroy(e);
  if (c->h_scal) cudaFreeHost(c->h_scal);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  delete c;
}

}  // extern "C"
