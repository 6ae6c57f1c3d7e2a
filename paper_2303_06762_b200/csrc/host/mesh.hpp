// Host-side mesh hierarchy for the hp-MG solve path (allowed on the host by
// the north star: "mesh hierarchy construction and assembly bookkeeping may
// stay on the host"). Numbering reproduces the reference exactly because it
// fixes the DOF layout and the multiplicative smoother order:
//   facets discovered in element order, local edge i = (v[i+1], v[i+2]),
//   facet direction lower -> higher vertex id      (reference inc/mesh.hpp:94-137)
//   red refinement: coarse vertices keep ids, midpoints appended in facet order,
//   children (v0,m2,m1) (m2,v1,m0) (m1,m0,v2) (m0,m1,m2) (inc/mesh.hpp:153-216)
// Storage is structure-of-arrays so that per-element geometry can be packed
// straight into device buffers.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <unordered_map>
#include <vector>

namespace hpmg {
namespace host {

enum : int { kTagInterior = 0, kTagDirichlet = 1, kTagOutflow = 2 };
enum : int8_t { kMedial = 0, kSkeleton = 1, kBoundaryChild = 2 };

struct TriMesh {
  std::vector<double> vx, vy;                 // vertex coordinates
  std::vector<std::array<int, 3>> ev;         // element vertices (ccw)
  std::vector<std::array<int, 3>> ef;         // facet opposite local vertex i
  std::vector<std::array<int8_t, 3>> esig;    // +1: global facet normal points outward
  std::vector<std::array<int8_t, 3>> erho;    // +1: local edge direction = global
  std::vector<int> fa, fb;                    // facet vertices, fa < fb
  std::vector<std::array<int, 2>> fe;         // adjacent elements, [1] = -1 on the boundary
  std::vector<int> ftag;

  int nv() const { return int(vx.size()); }
  int ne() const { return int(ev.size()); }
  int nf() const { return int(fa.size()); }

  double area(int e) const {
    const auto& v = ev[e];
    double ax = vx[v[1]] - vx[v[0]], ay = vy[v[1]] - vy[v[0]];
    double bx = vx[v[2]] - vx[v[0]], by = vy[v[2]] - vy[v[0]];
    return 0.5 * (ax * by - ay * bx);
  }
  double flen(int f) const {  // sqrt of the squared norm, as the reference's Vec2::norm
    double dx = vx[fb[f]] - vx[fa[f]], dy = vy[fb[f]] - vy[fa[f]];
    return std::sqrt(dx * dx + dy * dy);
  }
  void ftan(int f, double& tx, double& ty) const {
    double dx = vx[fb[f]] - vx[fa[f]], dy = vy[fb[f]] - vy[fa[f]];
    double l = std::sqrt(dx * dx + dy * dy);
    tx = dx / l;
    ty = dy / l;
  }
  void fnormal(int f, double& nx, double& ny) const {
    double tx, ty;
    ftan(f, tx, ty);
    nx = ty;
    ny = -tx;
  }
  void fmid(int f, double& x, double& y) const {
    x = 0.5 * (vx[fa[f]] + vx[fb[f]]);
    y = 0.5 * (vy[fa[f]] + vy[fb[f]]);
  }
  void fpoint(int f, double t, double& x, double& y) const {
    x = 0.5 * ((1.0 - t) * vx[fa[f]] + (1.0 + t) * vx[fb[f]]);
    y = 0.5 * ((1.0 - t) * vy[fa[f]] + (1.0 + t) * vy[fb[f]]);
  }

  /// Builds facets from elements; `keep_tags` carries over the tags of
  /// facets that existed before (matched by vertex pair).
  void build_facets(const std::unordered_map<uint64_t, int>* keep_tags = nullptr) {
    // facets numbered by first appearance (element order, local edge order):
    // the numbering fixes the DOF layout and the Gauss-Seidel order. Edges are
    // found in per-vertex buckets (CSR over the lower vertex, sized by the
    // number of element edges it starts) instead of a hash map.
    fa.clear(); fb.clear(); fe.clear(); ftag.clear();
    ef.assign(ne(), {0, 0, 0});
    const int nvv = nv();
    std::vector<int> start(size_t(nvv) + 1, 0);
    for (int e = 0; e < ne(); ++e)
      for (int i = 0; i < 3; ++i) {
        const int a = ev[e][(i + 1) % 3], b = ev[e][(i + 2) % 3];
        ++start[size_t(a < b ? a : b) + 1];
      }
    for (int v = 0; v < nvv; ++v) start[v + 1] += start[v];
    const size_t nslots = size_t(start[nvv]);
    std::vector<int> bhi(nslots), bid(nslots), used(size_t(nvv), 0);
    fa.reserve(size_t(ne()) * 2);
    fb.reserve(size_t(ne()) * 2);
    fe.reserve(size_t(ne()) * 2);
    ftag.reserve(size_t(ne()) * 2);
    for (int e = 0; e < ne(); ++e)
      for (int i = 0; i < 3; ++i) {
        int a = ev[e][(i + 1) % 3], b = ev[e][(i + 2) % 3];
        int lo = a < b ? a : b, hi = a < b ? b : a;
        const int s0 = start[lo], cnt = used[lo];
        int id = -1;
        for (int j = s0; j < s0 + cnt; ++j)
          if (bhi[j] == hi) {
            id = bid[j];
            break;
          }
        if (id < 0) {
          id = nf();
          bhi[size_t(s0 + cnt)] = hi;
          bid[size_t(s0 + cnt)] = id;
          ++used[lo];
          fa.push_back(lo);
          fb.push_back(hi);
          fe.push_back({e, -1});
          ftag.push_back(kTagInterior);
        } else {
          fe[id][1] = e;
        }
        ef[e][i] = id;
      }
    for (int f = 0; f < nf(); ++f) {
      if (fe[f][1] < 0) ftag[f] = kTagDirichlet;
      if (keep_tags) {
        uint64_t key = (uint64_t(uint32_t(fa[f])) << 32) | uint32_t(fb[f]);
        auto it = keep_tags->find(key);
        if (it != keep_tags->end()) ftag[f] = it->second;
      }
    }
    esig.assign(ne(), {0, 0, 0});
    erho.assign(ne(), {0, 0, 0});
    for (int e = 0; e < ne(); ++e) {
      const auto& v = ev[e];
      double cx = (vx[v[0]] + vx[v[1]] + vx[v[2]]) / 3.0, cy = (vy[v[0]] + vy[v[1]] + vy[v[2]]) / 3.0;
      for (int i = 0; i < 3; ++i) {
        int a = v[(i + 1) % 3], b = v[(i + 2) % 3];
        erho[e][i] = a < b ? 1 : -1;
        int f = ef[e][i];
        double mx, my, nx, ny;
        fmid(f, mx, my);
        fnormal(f, nx, ny);
        esig[e][i] = ((mx - cx) * nx + (my - cy) * ny) > 0.0 ? 1 : -1;
      }
    }
  }

  std::unordered_map<uint64_t, int> tag_map() const {
    std::unordered_map<uint64_t, int> m;
    for (int f = 0; f < nf(); ++f) m[(uint64_t(uint32_t(fa[f])) << 32) | uint32_t(fb[f])] = ftag[f];
    return m;
  }
};

/// Parent/child maps of one red refinement.
struct Refinement {
  std::vector<std::array<int, 4>> children;   // per coarse element
  std::vector<int> elem_parent;               // per fine element
  std::vector<int8_t> fclass;                 // per fine facet: kMedial/kSkeleton/kBoundaryChild
  std::vector<int> parent_facet;              // per fine facet, -1 for medial
  std::vector<int> parent_elem;               // per fine facet
  std::vector<std::array<int, 2>> fchildren;  // per coarse facet
};

inline TriMesh refine(const TriMesh& c, Refinement& R) {
  TriMesh f;
  f.vx = c.vx;
  f.vy = c.vy;
  const int nvc = c.nv();
  for (int k = 0; k < c.nf(); ++k) {
    double x, y;
    c.fmid(k, x, y);
    f.vx.push_back(x);
    f.vy.push_back(y);
  }
  R.children.resize(c.ne());
  R.elem_parent.resize(size_t(4) * c.ne());
  f.ev.reserve(size_t(4) * c.ne());
  for (int e = 0; e < c.ne(); ++e) {
    int v0 = c.ev[e][0], v1 = c.ev[e][1], v2 = c.ev[e][2];
    int m0 = nvc + c.ef[e][0], m1 = nvc + c.ef[e][1], m2 = nvc + c.ef[e][2];
    int base = f.ne();
    f.ev.push_back({v0, m2, m1});
    f.ev.push_back({m2, v1, m0});
    f.ev.push_back({m1, m0, v2});
    f.ev.push_back({m0, m1, m2});
    R.children[e] = {base, base + 1, base + 2, base + 3};
    for (int q = 0; q < 4; ++q) R.elem_parent[base + q] = e;
  }
  f.build_facets(nullptr);  // tags are inherited from parent facets below
  R.fclass.assign(f.nf(), kMedial);
  R.parent_facet.assign(f.nf(), -1);
  R.parent_elem.assign(f.nf(), -1);
  R.fchildren.assign(c.nf(), {-1, -1});
  for (int k = 0; k < f.nf(); ++k) {
    bool ac = f.fa[k] < nvc, bc = f.fb[k] < nvc;
    R.parent_elem[k] = R.elem_parent[f.fe[k][0]];
    if (ac == bc) {
      f.ftag[k] = kTagInterior;
      continue;
    }
    int cv = ac ? f.fa[k] : f.fb[k], mid = ac ? f.fb[k] : f.fa[k];
    int pf = mid - nvc;
    R.parent_facet[k] = pf;
    R.fclass[k] = c.fe[pf][1] < 0 ? kBoundaryChild : kSkeleton;
    f.ftag[k] = c.ftag[pf];
    R.fchildren[pf][cv == c.fa[pf] ? 0 : 1] = k;
  }
  return f;
}

/// n x n cells, diagonal (v00, v11) (reference inc/mesh.hpp:220-238).
inline TriMesh unit_square(int n) {
  TriMesh m;
  for (int j = 0; j <= n; ++j)
    for (int i = 0; i <= n; ++i) {
      m.vx.push_back(double(i) / n);
      m.vy.push_back(double(j) / n);
    }
  auto id = [n](int i, int j) { return j * (n + 1) + i; };
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      m.ev.push_back({id(i, j), id(i + 1, j), id(i + 1, j + 1)});
      m.ev.push_back({id(i, j), id(i + 1, j + 1), id(i, j + 1)});
    }
  m.build_facets();
  return m;
}

/// Backward-facing step, outflow on x = 4 (reference inc/mesh.hpp:243-279).
inline TriMesh step_domain(int n) {
  TriMesh m;
  const int nx = 4 * n, ny = n;
  std::vector<int> vid(size_t(nx + 1) * (ny + 1), -1);
  auto vert = [&](int i, int j) {
    int& id = vid[size_t(j) * (nx + 1) + i];
    if (id < 0) {
      id = m.nv();
      m.vx.push_back(double(i) / n);
      m.vy.push_back(double(j) / n);
    }
    return id;
  };
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      double cx = (i + 0.5) / n, cy = (j + 0.5) / n;
      if (!(cy > 0.5 || cx > 0.5)) continue;
      int a = vert(i, j), b = vert(i + 1, j), c = vert(i + 1, j + 1), d = vert(i, j + 1);
      m.ev.push_back({a, b, c});
      m.ev.push_back({a, c, d});
    }
  m.build_facets();
  for (int f = 0; f < m.nf(); ++f) {
    double x, y;
    m.fmid(f, x, y);
    if (m.ftag[f] != kTagInterior && std::abs(x - 4.0) < 1e-12) m.ftag[f] = kTagOutflow;
  }
  return m;
}

}  // namespace host
}  // namespace hpmg
