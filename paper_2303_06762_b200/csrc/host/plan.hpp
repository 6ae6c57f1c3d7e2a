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
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <memory>
#include <utility>
#include <vector>

#include "../kernels/condense.cuh"
#include "mesh.hpp"

namespace hpmg {
namespace host {

constexpr int kSlots = 5;      // self + 4 neighbours: a facet touches <= 2 triangles
constexpr int kMaxPatchF = 8;  // facets per vertex patch supported by the kernels
constexpr int kSmallPass = 24; // patches per pass of the one-CTA level kernel (small_levels.cu kPass)

using Field = std::function<void(double x, double y, double* out2)>;

/// Static-chunked parallel loop over [0, n) on up to 16 host threads (setup);
/// the first exception thrown by any iteration is rethrown after the join.
template <class F>
inline void parallel_for(int n, F&& f) {
  const int nt = std::max(1, std::min<int>({16, int(std::thread::hardware_concurrency()), n / 2048 + 1}));
  if (nt == 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::exception_ptr err;
  std::mutex mu;
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      try {
        const int a = int(int64_t(n) * t / nt), b = int(int64_t(n) * (t + 1) / nt);
        for (int i = a; i < b; ++i) f(i);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

/// std::allocator whose value-initialisation (resize) leaves elements
/// uninitialised: the large index/value arrays below are filled in parallel,
/// which also spreads their first-touch page faults over the threads.
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};
template <class T>
using BigVec = std::vector<T, NoInitAlloc<T>>;

/// Compressed adjacency built from (key, value) pairs in input order.
struct Csr32 {
  std::vector<int> ptr, val;
  const int* begin(int i) const { return val.data() + ptr[i]; }
  const int* end(int i) const { return val.data() + ptr[i + 1]; }
};

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
  BigVec<int> cols;                   // [nb][kSlots] block columns, -1 = empty
  // assembly gather per (row, slot): up to two (element, local row facet, local col facet)
  BigVec<int> gath;                   // [nb][kSlots][2][3]
  BigVec<int> row_elems;              // [nb][2][2] (element, local facet) ascending element
  // vertex patches (ascending vertex id, empty ones dropped)
  int npatch = 0, max_patch_f = 0;
  std::vector<int> patch_nf;          // facets per patch
  std::vector<int> patch_fac;         // [npatch][kMaxPatchF] block ids, ascending facet id
  std::vector<int64_t> inv_off;       // offset of each patch inverse (see set_inverse_layout)
  int64_t inv_total = 0;              // doubles stored
  int64_t inv_full_total = 0;         // sum np^2 (reference storage accounting)
  bool packed = true;
  std::vector<int> wave_ptr, wave_patch;  // forward wave order (balanced, see make_level)
  std::vector<int> asap_sizes;        // wave sizes of the as-soon-as-possible levelling
  std::vector<int> facet_patches;     // [nb][2] the two patches holding a block, ascending
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
  // uninitialised, each row's slots set to -1 by its own thread below (a
  // serial fill of these ~30 MB cost more than the rest of the plan)
  L.cols.resize(size_t(L.nb) * kSlots);
  L.gath.resize(size_t(L.nb) * kSlots * 6);
  L.row_elems.resize(size_t(L.nb) * 4);
  parallel_for(L.nb, [&](int r) {
    std::fill_n(&L.cols[size_t(r) * kSlots], kSlots, -1);
    std::fill_n(&L.gath[size_t(r) * kSlots * 6], kSlots * 6, -1);
    std::fill_n(&L.row_elems[size_t(r) * 4], 4, -1);
    const int f = L.block_facet[r];
    int nbv[6], nnb = 0;  // facets of the <= 2 elements of f, then sorted unique
    int slot_e = 0;
    for (int s = 0; s < 2; ++s) {
      const int e = m.fe[f][s];
      if (e < 0) continue;
      // ascending element order for deterministic sums
      slot_e++;
      for (int lf = 0; lf < 3; ++lf) {
        int g = L.facet_block[m.ef[e][lf]];
        if (g >= 0) nbv[nnb++] = g;
      }
    }
    std::sort(nbv, nbv + nnb);
    nnb = int(std::unique(nbv, nbv + nnb) - nbv);
    if (nnb > kSlots) throw std::runtime_error("facet couples to more than 5 facets");
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
    for (int s = 0; s < nnb; ++s) {
      const int c = nbv[s];
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
  });
  // vertex patches: facets incident to each vertex in facet order (inc/mesh.hpp:301-308)
  Csr32 vp;  // vertex -> incident facets (ascending facet id)
  Csr32 nbr;  // vertex -> mesh neighbours (the other end of those facets)
  vp.ptr.assign(m.nv() + 1, 0);
  for (int f = 0; f < m.nf(); ++f) {
    ++vp.ptr[m.fa[f] + 1];
    ++vp.ptr[m.fb[f] + 1];
  }
  for (int v = 0; v < m.nv(); ++v) vp.ptr[v + 1] += vp.ptr[v];
  vp.val.resize(vp.ptr[m.nv()]);
  nbr.ptr = vp.ptr;
  nbr.val.resize(vp.val.size());
  {
    std::vector<int> at(vp.ptr.begin(), vp.ptr.end() - 1);
    for (int f = 0; f < m.nf(); ++f) {
      const int a = at[m.fa[f]]++, b = at[m.fb[f]]++;
      vp.val[a] = f;
      nbr.val[a] = m.fb[f];
      vp.val[b] = f;
      nbr.val[b] = m.fa[f];
    }
  }
  std::vector<int> vertex_patch(m.nv(), -1);
  L.facet_patches.assign(size_t(L.nb) * 2, -1);
  L.patch_nf.reserve(m.nv());
  L.patch_fac.reserve(size_t(m.nv()) * kMaxPatchF);
  for (int v = 0; v < m.nv(); ++v) {
    int blocks[kMaxPatchF], nblk = 0;
    for (const int* fp = vp.begin(v); fp != vp.end(v); ++fp)
      if (L.facet_block[*fp] >= 0) {
        if (nblk == kMaxPatchF) throw std::runtime_error("vertex patch larger than supported");
        blocks[nblk++] = L.facet_block[*fp];
      }
    if (nblk == 0) continue;
    const int p = L.npatch++;
    vertex_patch[v] = p;
    L.patch_nf.push_back(nblk);
    L.max_patch_f = std::max(L.max_patch_f, nblk);
    for (int q = 0; q < kMaxPatchF; ++q) L.patch_fac.push_back(q < nblk ? blocks[q] : -1);
    for (int bi = 0; bi < nblk; ++bi) {
      const int b = blocks[bi];
      int* fp = &L.facet_patches[size_t(b) * 2];
      if (fp[0] < 0) fp[0] = p;
      else fp[1] = p;
    }
  }
  // exact wave schedule of the ascending-vertex sweep: depth(v) = 1 + max depth
  // of mesh neighbours u < v owning a patch. Same-depth
  // patches share no DOF and no operator coupling.
  std::vector<int> depth(m.nv(), -1);
  int maxd = -1;
  for (int v = 0; v < m.nv(); ++v) {
    if (vertex_patch[v] < 0) continue;
    int d = 0;
    for (const int* up = nbr.begin(v); up != nbr.end(v); ++up)
      if (*up < v && vertex_patch[*up] >= 0) d = std::max(d, depth[*up] + 1);
    depth[v] = d;
    maxd = std::max(maxd, d);
  }
  // Levelling. Any assignment with wave(u) < wave(v) for every coupled pair
  // u < v reproduces the sequential sweep exactly (every patch reads the same
  // x), so the as-soon-as-possible depths above fix only the wave count. On
  // wide schedules (9 waves, multi-CTA launches) the depths are used as they
  // are: re-levelling the 256^2 head towards even waves measured slower on
  // B200 (head sweeps 0.203 -> 0.208 ms). On narrow ones (> 12 waves: the
  // one-CTA level) every wave is capped at one pass of that kernel
  // (kSmallPass patches), placing patches from the last vertex down in the
  // latest wave of [depth, earliest successor wave - 1] below the cap: level
  // 1 of a 16x16 base goes from 66 to 50 passes per sweep.
  const int nw = maxd + 1;
  L.asap_sizes.assign(nw, 0);
  for (int v = 0; v < m.nv(); ++v)
    if (vertex_patch[v] >= 0) L.asap_sizes[depth[v]]++;
  const bool narrow = nw > 12;
  const int cap = kSmallPass;
  // narrow: placement in descending vertex order (successors first), latest
  // wave of [depth, earliest successor wave - 1] below the cap, else the least loaded
  std::vector<int> wave_of_v(m.nv(), -1), load(nw, 0);
  for (int v = m.nv() - 1; v >= 0; --v) {
    if (vertex_patch[v] < 0) continue;
    int w = depth[v];
    if (narrow) {
      int hi = maxd;
      for (const int* up = nbr.begin(v); up != nbr.end(v); ++up)
        if (*up > v && vertex_patch[*up] >= 0) hi = std::min(hi, wave_of_v[*up] - 1);
      const int lo = depth[v];
      if (lo > hi) throw std::logic_error("wave levelling: empty placement range");
      w = -1;
      for (int c = hi; c >= lo && w < 0; --c)
        if (load[c] < cap) w = c;
      if (w < 0) {
        w = hi;
        for (int c = hi - 1; c >= lo; --c)
          if (load[c] < load[w]) w = c;
      }
    }
    wave_of_v[v] = w;
    load[w]++;
  }
  std::vector<std::vector<int>> waves(nw);
  for (int v = 0; v < m.nv(); ++v)
    if (vertex_patch[v] >= 0) waves[wave_of_v[v]].push_back(vertex_patch[v]);
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
