// Host bookkeeping for one multigrid level: free-facet block numbering, the
// fixed-width block-sparse (ELL-BSR) pattern, the deterministic assembly
// gather lists, vertex patches with their exact parallel wave schedule,
// element geometry packing and the CR-GMG averaging transfer pattern.
//
// Device layout: a level with order k has block size bs = 2(k+1);
// block row f is the f-th free facet in ascending mesh-facet order and holds
// [flux_0, tang_0, flux_1, tang_1, ...] (the reference patch order,
// inc/smoother.hpp:13-28). The reference free order (all flux modes, then all
// tangential modes, inc/fespace.hpp:343-347, 508-513) is a pure permutation of
// it: flux (f,i) -> f*(k+1)+i, tang (f,i) -> nb*(k+1) + f*(k+1)+i.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <functional>
#include <vector>

#include "../kernels/condense.cuh"
#include "mesh.hpp"

namespace hpmg {
namespace host {

constexpr int kSlots = 5;      // self + 4 neighbours: a facet touches <= 2 triangles
constexpr int kMaxPatchF = 8;  // facets per vertex patch supported by the kernels

using Field = std::function<void(double x, double y, double* out2)>;

/// Reference edge lengths: edge 0 = (1,0)-(0,1), edges 1, 2 unit.
inline double ref_edge_len(int le) { return le == 0 ? std::sqrt(2.0) : 1.0; }

inline ElemGeo element_geometry(const TriMesh& m, int e) {
  ElemGeo g{};
  const auto& v = m.ev[e];
  const double x0 = m.vx[v[0]], y0 = m.vy[v[0]];
  g.J[0] = m.vx[v[1]] - x0;
  g.J[2] = m.vy[v[1]] - y0;
  g.J[1] = m.vx[v[2]] - x0;
  g.J[3] = m.vy[v[2]] - y0;
  g.detJ = g.J[0] * g.J[3] - g.J[1] * g.J[2];
  g.Ji[0] = g.J[3] / g.detJ;
  g.Ji[1] = -g.J[1] / g.detJ;
  g.Ji[2] = -g.J[2] / g.detJ;
  g.Ji[3] = g.J[0] / g.detJ;
  for (int le = 0; le < 3; ++le) {
    const int f = m.ef[e][le];
    const double len = m.flen(f);
    g.fac[le] = double(m.esig[e][le]) * len / ref_edge_len(le);
    g.rho[le] = double(m.erho[e][le]);
    double nx, ny, tx, ty;
    m.fnormal(f, nx, ny);
    m.ftan(f, tx, ty);
    g.n[2 * le] = double(m.esig[e][le]) * nx;
    g.n[2 * le + 1] = double(m.esig[e][le]) * ny;
    g.tf[2 * le] = tx;
    g.tf[2 * le + 1] = ty;
    g.ds[le] = 0.5 * len;
  }
  return g;
}

struct LevelPlan {
  int k = 0, bs = 2, nfd = 1;
  const TriMesh* mesh = nullptr;
  int nb = 0;                         // free facets = block rows
  std::vector<int> block_facet;       // block -> mesh facet
  std::vector<int> facet_block;       // mesh facet -> block or -1 (Dirichlet)
  std::vector<int> cols;              // [nb][kSlots] block columns, -1 = empty
  // assembly gather per (row, slot): up to two (element, local row facet, local col facet)
  std::vector<int> gath;              // [nb][kSlots][2][3]
  std::vector<int> row_elems;         // [nb][2][2] (element, local facet) ascending element
  // vertex patches (ascending vertex id, empty ones dropped)
  int npatch = 0, max_patch_f = 0;
  std::vector<int> patch_nf;          // facets per patch
  std::vector<int> patch_fac;         // [npatch][kMaxPatchF] block ids, ascending facet id
  std::vector<int64_t> inv_off;       // offset of each patch inverse (see set_inverse_layout)
  int64_t inv_total = 0;              // doubles stored
  int64_t inv_full_total = 0;         // sum np^2 (reference storage accounting)
  bool packed = true;
  std::vector<int> wave_ptr, wave_patch;  // forward wave order
  std::vector<int> facet_patches;     // [nb][2] the two patches holding a block, ascending
  // dataflow sweep: patches of the mesh neighbours of each patch's vertex
  // (renumbered ids; the forward sweep waits on the smaller, the reverse on the larger)
  int max_dep = 0;
  std::vector<int> patch_ndep;        // [npatch]
  std::vector<int> patch_dep;         // [npatch][max_dep], -1 padded
  int nwaves() const { return int(wave_ptr.size()) - 1; }
  int64_t n() const { return int64_t(nb) * bs; }
};

inline void set_inverse_layout(LevelPlan& L, bool packed);

/// Free blocks, ELL pattern, gather lists, patches and waves for one level.
inline LevelPlan make_level(const TriMesh& m, int k) {
  LevelPlan L;
  L.k = k;
  L.nfd = k + 1;
  L.bs = 2 * (k + 1);
  L.mesh = &m;
  L.facet_block.assign(m.nf(), -1);
  for (int f = 0; f < m.nf(); ++f)
    if (m.ftag[f] != kTagDirichlet) {
      L.facet_block[f] = L.nb++;
      L.block_facet.push_back(f);
    }
  // ELL pattern: facets sharing an element with the row facet, sorted
  L.cols.assign(size_t(L.nb) * kSlots, -1);
  L.gath.assign(size_t(L.nb) * kSlots * 6, -1);
  L.row_elems.assign(size_t(L.nb) * 4, -1);
  for (int r = 0; r < L.nb; ++r) {
    const int f = L.block_facet[r];
    std::vector<int> nb;
    int slot_e = 0;
    for (int s = 0; s < 2; ++s) {
      const int e = m.fe[f][s];
      if (e < 0) continue;
      // ascending element order for deterministic sums
      slot_e++;
      for (int lf = 0; lf < 3; ++lf) {
        int g = L.facet_block[m.ef[e][lf]];
        if (g >= 0) nb.push_back(g);
      }
    }
    std::sort(nb.begin(), nb.end());
    nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    if (int(nb.size()) > kSlots) throw std::runtime_error("facet couples to more than 5 facets");
    std::array<int, 2> es = {m.fe[f][0], m.fe[f][1]};
    if (es[1] >= 0 && es[1] < es[0]) std::swap(es[0], es[1]);
    int re = 0;
    for (int e : es) {
      if (e < 0) continue;
      int lf = -1;
      for (int q = 0; q < 3; ++q)
        if (m.ef[e][q] == f) lf = q;
      L.row_elems[size_t(r) * 4 + 2 * re] = e;
      L.row_elems[size_t(r) * 4 + 2 * re + 1] = lf;
      ++re;
    }
    for (size_t s = 0; s < nb.size(); ++s) {
      const int c = nb[s];
      L.cols[size_t(r) * kSlots + s] = c;
      const int gf = L.block_facet[c];
      int cnt = 0;
      for (int e : es) {
        if (e < 0) continue;
        int la = -1, lb = -1;
        for (int q = 0; q < 3; ++q) {
          if (m.ef[e][q] == f) la = q;
          if (m.ef[e][q] == gf) lb = q;
        }
        if (la < 0 || lb < 0) continue;
        int* gp = &L.gath[(size_t(r) * kSlots + s) * 6 + 3 * cnt];
        gp[0] = e;
        gp[1] = la;
        gp[2] = lb;
        ++cnt;
      }
    }
    (void)slot_e;
  }
  // vertex patches: facets incident to each vertex in facet order (inc/mesh.hpp:301-308)
  std::vector<std::vector<int>> vp(m.nv());
  for (int f = 0; f < m.nf(); ++f) {
    vp[m.fa[f]].push_back(f);
    vp[m.fb[f]].push_back(f);
  }
  std::vector<int> vertex_patch(m.nv(), -1);
  L.facet_patches.assign(size_t(L.nb) * 2, -1);
  for (int v = 0; v < m.nv(); ++v) {
    std::vector<int> blocks;
    for (int f : vp[v])
      if (L.facet_block[f] >= 0) blocks.push_back(L.facet_block[f]);
    if (blocks.empty()) continue;
    if (int(blocks.size()) > kMaxPatchF) throw std::runtime_error("vertex patch larger than supported");
    const int p = L.npatch++;
    vertex_patch[v] = p;
    L.patch_nf.push_back(int(blocks.size()));
    L.max_patch_f = std::max(L.max_patch_f, int(blocks.size()));
    for (int q = 0; q < kMaxPatchF; ++q) L.patch_fac.push_back(q < int(blocks.size()) ? blocks[q] : -1);
    for (int b : blocks) {
      int* fp = &L.facet_patches[size_t(b) * 2];
      if (fp[0] < 0) fp[0] = p;
      else fp[1] = p;
    }
  }
  // exact wave schedule of the ascending-vertex sweep: depth(v) = 1 + max depth
  // of mesh neighbours u < v owning a patch. Same-depth
  // patches share no DOF and no operator coupling.
  std::vector<std::vector<int>> nbr(m.nv());
  for (int f = 0; f < m.nf(); ++f) {
    nbr[m.fa[f]].push_back(m.fb[f]);
    nbr[m.fb[f]].push_back(m.fa[f]);
  }
  std::vector<int> depth(m.nv(), -1);
  int maxd = -1;
  for (int v = 0; v < m.nv(); ++v) {
    if (vertex_patch[v] < 0) continue;
    int d = 0;
    for (int u : nbr[v])
      if (u < v && vertex_patch[u] >= 0) d = std::max(d, depth[u] + 1);
    depth[v] = d;
    maxd = std::max(maxd, d);
  }
  std::vector<std::vector<int>> waves(maxd + 1);
  for (int v = 0; v < m.nv(); ++v)
    if (vertex_patch[v] >= 0) waves[depth[v]].push_back(vertex_patch[v]);
  L.wave_ptr.push_back(0);
  for (auto& w : waves) {
    for (int p : w) L.wave_patch.push_back(p);
    L.wave_ptr.push_back(int(L.wave_patch.size()));
  }
  // Renumber patches in wave order so that a wave is a contiguous patch
  // range on the device (no wave -> patch indirection in the sweep kernels).
  // facet_patches keeps the reference's ascending-vertex order of the two
  // patches of a facet (the additive smoother sums in that order).
  std::vector<int> newid(L.npatch);
  for (int q = 0; q < L.npatch; ++q) newid[L.wave_patch[q]] = q;
  std::vector<int> nf2(L.npatch), fac2(L.patch_fac.size());
  for (int p = 0; p < L.npatch; ++p) {
    nf2[newid[p]] = L.patch_nf[p];
    for (int q = 0; q < kMaxPatchF; ++q) fac2[size_t(newid[p]) * kMaxPatchF + q] = L.patch_fac[size_t(p) * kMaxPatchF + q];
  }
  L.patch_nf.swap(nf2);
  L.patch_fac.swap(fac2);
  for (auto& fp : L.facet_patches)
    if (fp >= 0) fp = newid[fp];
  {
    std::vector<std::vector<int>> dep(L.npatch);
    for (int v = 0; v < m.nv(); ++v) {
      if (vertex_patch[v] < 0) continue;
      auto& d = dep[newid[vertex_patch[v]]];
      for (int u : nbr[v])
        if (vertex_patch[u] >= 0) d.push_back(newid[vertex_patch[u]]);
      std::sort(d.begin(), d.end());
      d.erase(std::unique(d.begin(), d.end()), d.end());
      L.max_dep = std::max(L.max_dep, int(d.size()));
    }
    L.patch_ndep.assign(L.npatch, 0);
    L.patch_dep.assign(size_t(L.npatch) * std::max(L.max_dep, 1), -1);
    for (int p = 0; p < L.npatch; ++p) {
      L.patch_ndep[p] = int(dep[p].size());
      for (size_t i = 0; i < dep[p].size(); ++i) L.patch_dep[size_t(p) * L.max_dep + i] = dep[p][i];
    }
  }
  for (int q = 0; q < L.npatch; ++q) L.wave_patch[q] = q;
  set_inverse_layout(L, true);
  return L;
}

/// Offsets of the per-patch explicit inverses: packed lower triangle by
/// columns (np(np+1)/2 doubles) for symmetric operators, full column-major
/// (np^2) otherwise.
inline void set_inverse_layout(LevelPlan& L, bool packed) {
  L.packed = packed;
  L.inv_off.assign(L.npatch, 0);
  L.inv_total = 0;
  L.inv_full_total = 0;
  for (int p = 0; p < L.npatch; ++p) {
    const int64_t np = int64_t(L.patch_nf[p]) * L.bs;
    L.inv_off[p] = L.inv_total;
    L.inv_total += packed ? ((np * (np + 1) / 2 + 1) & ~int64_t(1)) : np * np;  // even: 16-byte TMA rows
    L.inv_full_total += np * np;
  }
}

}  // namespace host
}  // namespace hpmg
