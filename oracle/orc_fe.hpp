// TEST INFRASTRUCTURE ONLY (see orc_core.hpp). Hierarchical RT_k reference
// basis, per-order tables, compound skeleton DOF map, element geometry,
// interpolation and Dirichlet constraints (reference inc/fespace.hpp).
#pragma once

#include <map>
#include <memory>
#include <mutex>

#include "orc_mesh.hpp"

namespace orc {

struct RefEdge {
  V2 a, b, n_out;
  Real len;
};

/// Reference triangle edges with outward normals (inc/fespace.hpp:27-42).
inline const std::array<RefEdge, 3>& ref_edges() {
  static const std::array<RefEdge, 3> e = [] {
    const V2 v[3] = {{0, 0}, {1, 0}, {0, 1}};
    std::array<RefEdge, 3> out{};
    for (int i = 0; i < 3; ++i) {
      V2 a = v[(i + 1) % 3], b = v[(i + 2) % 3];
      V2 t = (b - a).normalized();
      V2 n(t.y, -t.x);
      if (n.dot(a - v[i]) < 0) n = n * -1.0;
      out[i] = RefEdge{a, b, n, (b - a).norm()};
    }
    return out;
  }();
  return e;
}

struct RTRef {
  int k = 0, n_facet = 1, n_bubble = 0, n_div = 0, dim = 3;
  std::vector<std::array<Poly, 2>> val;
  std::vector<std::array<Poly, 4>> jac;
  std::vector<Poly> div;
  int facet_fn(int e, int i) const { return e * n_facet + i; }
  int interior_fn(int j) const { return 3 * n_facet + j; }
  int n_interior() const { return n_bubble + n_div; }
};

/// Builds the hierarchical RT_k basis: RT0 facet functions, facet functions
/// i>=1 from a square constrained solve, divergence-free bubbles and
/// divergence-reproducing interior functions (inc/fespace.hpp:114-228).
/// Highest order accepted: 3 as in the reference (inc/fespace.hpp:115); tests
/// of the device path beyond the reference raise it (orc_set_max_order), the
/// construction itself being order-generic.
inline int& max_order() {
  static int m = 3;
  return m;
}

inline RTRef build_rt(int k) {
  if (k < 0 || k > max_order())
    throw std::invalid_argument(max_order() == 3 ? "order k must be in 0..3" : "order k out of range");
  RTRef rt;
  rt.k = k;
  rt.n_facet = k + 1;
  const int ns = Poly::dim(k);
  rt.n_div = ns - 1;
  rt.n_bubble = k * (k + 1) - rt.n_div;
  rt.dim = 3 * rt.n_facet + rt.n_bubble + rt.n_div;

  // generic family spanning RT_k (inc/fespace.hpp:73-86)
  std::vector<Poly> q = orthonormal_basis(k);
  std::vector<std::array<Poly, 2>> gen;
  for (const Poly& s : q) {
    gen.push_back({s, Poly(0)});
    gen.push_back({Poly(0), s});
  }
  for (int j = 0; j <= k; ++j) {
    Poly m = Poly::mono(k - j, j);
    gen.push_back({Poly::mono(1, 0) * m, Poly::mono(0, 1) * m});
  }
  const int gd = int(gen.size());
  std::vector<Poly> gdiv(gd);
  for (int g = 0; g < gd; ++g) gdiv[g] = gen[g][0].dx() + gen[g][1].dy();
  const auto& E = ref_edges();

  // facet Legendre moments (inc/fespace.hpp:90-110)
  Mat M(3 * (k + 1), gd);
  {
    LineRule lr = line_rule(2 * k + 3);
    Real leg[8];
    for (int e = 0; e < 3; ++e)
      for (std::size_t qp = 0; qp < lr.pts.size(); ++qp) {
        Real t = lr.pts[qp];
        V2 x = (E[e].a * (1.0 - t) + E[e].b * (1.0 + t)) * 0.5;
        legendre_all(k, t, leg);
        for (int g = 0; g < gd; ++g) {
          Real vn = gen[g][0].eval(x.x, x.y) * E[e].n_out.x + gen[g][1].eval(x.x, x.y) * E[e].n_out.y;
          for (int i = 0; i <= k; ++i) M(e * (k + 1) + i, g) += 0.5 * (2 * i + 1) * lr.wts[qp] * vn * leg[i];
        }
      }
  }
  Mat D(rt.n_div, gd);
  for (int p = 1; p < ns; ++p)
    for (int g = 0; g < gd; ++g) D(p - 1, g) = tri_l2(gdiv[g], q[p]);
  Mat G(gd, gd);
  for (int a = 0; a < gd; ++a)
    for (int b = a; b < gd; ++b) {
      G(a, b) = tri_l2(gen[a][0], gen[b][0]) + tri_l2(gen[a][1], gen[b][1]);
      G(b, a) = G(a, b);
    }

  Mat bubbles(gd, 0), psis(gd, 0);
  const int nk = k * (k + 1);
  if (nk > 0) {
    SVD svm(M);
    Mat W(gd, nk);
    for (int i = 0; i < gd; ++i)
      for (int j = 0; j < nk; ++j) W(i, j) = svm.V(i, gd - nk + j);
    Mat DW = matmul(D, W);
    SVD svd(DW);
    if (int(svd.s.size()) < rt.n_div || svd.s[rt.n_div - 1] < 1e-10)
      throw std::logic_error("interior divergence map is rank-deficient");
    Mat Vr(nk, rt.n_bubble);
    for (int i = 0; i < nk; ++i)
      for (int j = 0; j < rt.n_bubble; ++j) Vr(i, j) = svd.V(i, nk - rt.n_bubble + j);
    bubbles = matmul(W, Vr);
    for (int c = 0; c < rt.n_bubble; ++c) {
      Vec col(gd);
      for (int i = 0; i < gd; ++i) col[i] = bubbles(i, c);
      Real nrm = std::sqrt(dot(col, matvec(G, col)));
      for (int i = 0; i < gd; ++i) bubbles(i, c) /= nrm;
    }
    psis = Mat(gd, rt.n_div);
    for (int j = 0; j < rt.n_div; ++j) {
      Vec rhs(rt.n_div, 0.0);
      rhs[j] = 1.0;
      Vec y = svd.solve(rhs);
      Vec c = matvec(W, y);
      for (int i = 0; i < gd; ++i) psis(i, j) = c[i];
    }
  }

  const int nrows = 3 * (k + 1) + rt.n_div + rt.n_bubble;
  if (nrows != gd) throw std::logic_error("constraint count mismatch");
  Mat sys(nrows, gd);
  for (int i = 0; i < 3 * (k + 1); ++i)
    for (int g = 0; g < gd; ++g) sys(i, g) = M(i, g);
  for (int i = 0; i < rt.n_div; ++i)
    for (int g = 0; g < gd; ++g) sys(3 * (k + 1) + i, g) = D(i, g);
  if (rt.n_bubble > 0) {
    Mat BG = matmul(bubbles.t(), G);
    for (int i = 0; i < rt.n_bubble; ++i)
      for (int g = 0; g < gd; ++g) sys(3 * (k + 1) + rt.n_div + i, g) = BG(i, g);
  }
  FullLU lu(sys);
  if (!lu.invertible()) throw std::logic_error("facet constraint system is singular");

  rt.val.resize(rt.dim);
  rt.jac.resize(rt.dim);
  rt.div.resize(rt.dim);
  auto set_fn = [&rt](int f, const Poly& vx, const Poly& vy) {
    rt.val[f] = {vx, vy};
    rt.jac[f] = {vx.dx(), vx.dy(), vy.dx(), vy.dy()};
    rt.div[f] = vx.dx() + vy.dy();
  };
  auto combine = [&](const Vec& c, int f) {
    Poly fx(0), fy(0);
    for (int g = 0; g < gd; ++g) {
      if (c[g] == 0.0) continue;
      fx += c[g] * gen[g][0];
      fy += c[g] * gen[g][1];
    }
    set_fn(f, fx, fy);
  };
  const V2 vtx[3] = {{0, 0}, {1, 0}, {0, 1}};
  for (int e = 0; e < 3; ++e) {
    Poly vx = Poly::mono(1, 0), vy = Poly::mono(0, 1);
    vx -= vtx[e].x * Poly::mono(0, 0);
    vy -= vtx[e].y * Poly::mono(0, 0);
    set_fn(rt.facet_fn(e, 0), E[e].len * vx, E[e].len * vy);
    for (int i = 1; i <= k; ++i) {
      Vec rhs(nrows, 0.0);
      rhs[e * (k + 1) + i] = 1.0;
      Vec c = lu.solve(rhs);
      Vec res = matvec(sys, c);
      for (int r = 0; r < nrows; ++r) res[r] -= rhs[r];
      if (norm(res) > 1e-9) throw std::logic_error("facet basis solve failed");
      combine(c, rt.facet_fn(e, i));
    }
  }
  for (int j = 0; j < rt.n_bubble + rt.n_div; ++j) {
    Vec c(gd);
    for (int i = 0; i < gd; ++i) c[i] = j < rt.n_bubble ? bubbles(i, j) : psis(i, j - rt.n_bubble);
    combine(c, rt.interior_fn(j));
  }
  return rt;
}

/// Per-order basis tables at the volume/edge rules (inc/fespace.hpp:233-330).
struct RefData {
  int k = 0;
  RTRef rt;
  std::vector<Poly> scalar;
  TriRule vol;
  LineRule edge;
  // vol tables: [q][row][fn]
  std::vector<Mat> vval, vjac;  // 2 x dim, 4 x dim
  Mat vdiv;                      // nq x dim
  std::array<std::vector<Mat>, 3> eval_;  // per edge per point: 2 x dim
  Mat vscal;                     // nq x ns
  std::array<Mat, 3> escal;      // per edge: nqe x ns
  int nq() const { return int(vol.pts.size()); }
  int nqe() const { return int(edge.pts.size()); }
  int ns() const { return int(scalar.size()); }
};

inline const RefData& ref_data(int k) {
  static std::map<int, std::unique_ptr<RefData>> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(k);
  if (it != cache.end()) return *it->second;
  auto d = std::make_unique<RefData>();
  RefData& rd = *d;
  rd.k = k;
  rd.rt = build_rt(k);
  rd.scalar = orthonormal_basis(k);
  rd.vol = tri_rule(3 * k + 4);
  rd.edge = line_rule(3 * k + 4);
  const int dim = rd.rt.dim, ns = rd.ns(), nq = rd.nq();
  rd.vval.assign(nq, Mat(2, dim));
  rd.vjac.assign(nq, Mat(4, dim));
  rd.vdiv = Mat(nq, dim);
  rd.vscal = Mat(nq, ns);
  for (int q = 0; q < nq; ++q) {
    Real x = rd.vol.pts[q].x, y = rd.vol.pts[q].y;
    for (int f = 0; f < dim; ++f) {
      rd.vval[q](0, f) = rd.rt.val[f][0].eval(x, y);
      rd.vval[q](1, f) = rd.rt.val[f][1].eval(x, y);
      for (int c = 0; c < 4; ++c) rd.vjac[q](c, f) = rd.rt.jac[f][c].eval(x, y);
      rd.vdiv(q, f) = rd.rt.div[f].eval(x, y);
    }
    for (int s = 0; s < ns; ++s) rd.vscal(q, s) = rd.scalar[s].eval(x, y);
  }
  const auto& E = ref_edges();
  for (int e = 0; e < 3; ++e) {
    rd.eval_[e].assign(rd.nqe(), Mat(2, dim));
    rd.escal[e] = Mat(rd.nqe(), ns);
    for (int q = 0; q < rd.nqe(); ++q) {
      Real t = rd.edge.pts[q];
      V2 xp = (E[e].a * (1.0 - t) + E[e].b * (1.0 + t)) * 0.5;
      for (int f = 0; f < dim; ++f) {
        rd.eval_[e][q](0, f) = rd.rt.val[f][0].eval(xp.x, xp.y);
        rd.eval_[e][q](1, f) = rd.rt.val[f][1].eval(xp.x, xp.y);
      }
      for (int s = 0; s < ns; ++s) rd.escal[e](q, s) = rd.scalar[s].eval(xp.x, xp.y);
    }
  }
  auto ins = cache.emplace(k, std::move(d));
  return *ins.first->second;
}

/// Compound skeleton space: per facet k+1 flux then (separately) k+1
/// tangential Legendre coefficients (inc/fespace.hpp:335-356).
struct Space {
  const Mesh* mesh = nullptr;
  int k = 0;
  Space() = default;
  Space(const Mesh& m, int order) : mesh(&m), k(order) {}
  int nfd() const { return k + 1; }
  Index n_flux() const { return Index(mesh->nf()) * nfd(); }
  Index n_compound() const { return 2 * n_flux(); }
  Index flux(int f, int i) const { return Index(f) * nfd() + i; }
  Index tang(int f, int i) const { return n_flux() + Index(f) * nfd() + i; }
  int n_int() const { return k * (k + 1); }
  Index n_interior() const { return Index(mesh->ne()) * n_int(); }
  Index interior(int e, int j) const { return Index(e) * n_int() + j; }
};

/// Affine element map and facet orientation factors (inc/fespace.hpp:360-393).
struct Geo {
  Real J[2][2], Ji[2][2], detJ, area;
  V2 x0;
  int facet[3], sigma[3], rho[3];
  Real flen[3];
  Geo(const Mesh& m, int e) {
    const auto& E = m.el[e];
    x0 = m.vtx[E.v[0]];
    V2 c0 = m.vtx[E.v[1]] - x0, c1 = m.vtx[E.v[2]] - x0;
    J[0][0] = c0.x; J[1][0] = c0.y; J[0][1] = c1.x; J[1][1] = c1.y;
    detJ = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    Ji[0][0] = J[1][1] / detJ; Ji[0][1] = -J[0][1] / detJ;
    Ji[1][0] = -J[1][0] / detJ; Ji[1][1] = J[0][0] / detJ;
    area = 0.5 * detJ;
    for (int i = 0; i < 3; ++i) {
      facet[i] = E.facet[i];
      flen[i] = m.flen(E.facet[i]);
      sigma[i] = E.sigma[i];
      rho[i] = E.rho[i];
    }
  }
  V2 map(const V2& xh) const { return {x0.x + J[0][0] * xh.x + J[0][1] * xh.y, x0.y + J[1][0] * xh.x + J[1][1] * xh.y}; }
  V2 applyJ(Real a, Real b) const { return {J[0][0] * a + J[0][1] * b, J[1][0] * a + J[1][1] * b}; }
  Real rt_factor(int e, int i) const {
    Real f = Real(sigma[e]) * flen[e] / ref_edges()[e].len;
    return (i % 2 == 1 && rho[e] < 0) ? -f : f;
  }
};

struct RTField {
  Space V;
  Vec flux, interior;
};

/// RT_k interpolation: facet Legendre moments, interior by local L2 solve
/// (inc/fespace.hpp:404-461).
inline RTField interpolate_rt(const Mesh& mesh, int k, const Field& field) {
  const RefData& rd = ref_data(k);
  RTField out;
  out.V = Space(mesh, k);
  out.flux.assign(out.V.n_flux(), 0.0);
  out.interior.assign(out.V.n_interior(), 0.0);
  Real leg[8];
  for (int f = 0; f < mesh.nf(); ++f) {
    V2 n = mesh.fnormal(f);
    for (std::size_t q = 0; q < rd.edge.pts.size(); ++q) {
      Real t = rd.edge.pts[q];
      Real vn = field(mesh.fpoint(f, t)).dot(n);
      legendre_all(k, t, leg);
      for (int i = 0; i <= k; ++i) out.flux[out.V.flux(f, i)] += 0.5 * (2 * i + 1) * rd.edge.wts[q] * vn * leg[i];
    }
  }
  const int ni = out.V.n_int();
  if (ni == 0) return out;
  for (int e = 0; e < mesh.ne(); ++e) {
    Geo geo(mesh, e);
    Mat A(ni, ni);
    Vec b(ni, 0.0);
    for (int q = 0; q < rd.nq(); ++q) {
      Real w = rd.vol.wts[q] * geo.detJ;
      auto phys = [&](int fn) { return geo.applyJ(rd.vval[q](0, fn), rd.vval[q](1, fn)) / geo.detJ; };
      V2 gi = field(geo.map(rd.vol.pts[q]));
      for (int le = 0; le < 3; ++le)
        for (int i = 0; i <= k; ++i) {
          Real c = out.flux[out.V.flux(geo.facet[le], i)] * geo.rt_factor(le, i);
          gi -= phys(rd.rt.facet_fn(le, i)) * c;
        }
      for (int a = 0; a < ni; ++a) {
        V2 va = phys(rd.rt.interior_fn(a));
        b[a] += w * va.dot(gi);
        for (int c = 0; c < ni; ++c) A(a, c) += w * va.dot(phys(rd.rt.interior_fn(c)));
      }
    }
    Vec sol = LU(A).solve(b);
    for (int j = 0; j < ni; ++j) out.interior[out.V.interior(e, j)] = sol[j];
  }
  return out;
}

/// Full hybrid state (compound + interior) (reference inc/assembly.hpp:15-35).
struct HDGVel {
  Space V;
  Vec compound, interior;
  static HDGVel zero(const Space& s) {
    HDGVel u;
    u.V = s;
    u.compound.assign(s.n_compound(), 0.0);
    u.interior.assign(s.n_interior(), 0.0);
    return u;
  }
};

/// (reference inc/assembly.hpp:40-62)
inline HDGVel interpolate_hdg(const Mesh& mesh, int k, const Field& field) {
  RTField rt = interpolate_rt(mesh, k, field);
  HDGVel u;
  u.V = rt.V;
  u.compound.assign(u.V.n_compound(), 0.0);
  for (Index i = 0; i < u.V.n_flux(); ++i) u.compound[i] = rt.flux[i];
  u.interior = rt.interior;
  const LineRule& lr = ref_data(k).edge;
  Real leg[8];
  for (int f = 0; f < mesh.nf(); ++f) {
    V2 tau = mesh.ftan(f);
    for (std::size_t q = 0; q < lr.pts.size(); ++q) {
      Real t = lr.pts[q];
      Real vt = field(mesh.fpoint(f, t)).dot(tau);
      legendre_all(k, t, leg);
      for (int i = 0; i <= k; ++i) u.compound[u.V.tang(f, i)] += 0.5 * (2 * i + 1) * lr.wts[q] * vt * leg[i];
    }
  }
  return u;
}

/// Dirichlet constraints with boundary Legendre moments (inc/fespace.hpp:470-535).
struct Constraints {
  Index n_full = 0, n_free = 0;
  std::vector<Index> full_to_free, free_to_full;
  Vec g_full;
  static Constraints build(const Space& V, const Field& g) {
    const Mesh& m = *V.mesh;
    Constraints c;
    c.n_full = V.n_compound();
    c.full_to_free.assign(c.n_full, -1);
    c.g_full.assign(c.n_full, 0.0);
    std::vector<char> con(c.n_full, 0);
    const int k = V.k;
    LineRule lr = line_rule(2 * k + 6);
    Real leg[8];
    for (int f = 0; f < m.nf(); ++f) {
      if (m.fc[f].tag != kDirichlet) continue;
      for (int i = 0; i <= k; ++i) con[V.flux(f, i)] = con[V.tang(f, i)] = 1;
      if (!g) continue;
      V2 n = m.fnormal(f), tau = m.ftan(f);
      for (std::size_t q = 0; q < lr.pts.size(); ++q) {
        Real t = lr.pts[q];
        V2 gv = g(m.fpoint(f, t));
        legendre_all(k, t, leg);
        for (int i = 0; i <= k; ++i) {
          Real w = 0.5 * (2 * i + 1) * lr.wts[q] * leg[i];
          c.g_full[V.flux(f, i)] += w * gv.dot(n);
          c.g_full[V.tang(f, i)] += w * gv.dot(tau);
        }
      }
    }
    for (Index d = 0; d < c.n_full; ++d) {
      if (con[d]) continue;
      c.full_to_free[d] = Index(c.free_to_full.size());
      c.free_to_full.push_back(d);
    }
    c.n_free = Index(c.free_to_full.size());
    return c;
  }
  Vec to_free(const Vec& full) const {
    Vec o(n_free);
    for (Index i = 0; i < n_free; ++i) o[i] = full[free_to_full[i]];
    return o;
  }
  Vec to_full(const Vec& fr) const {
    Vec o = g_full;
    for (Index i = 0; i < n_free; ++i) o[free_to_full[i]] = fr[i];
    return o;
  }
};

}  // namespace orc
