// TEST INFRASTRUCTURE ONLY (see orc_core.hpp). CPU restatement of the
// reference's post-processing and error measurement (inc/postprocess.hpp:16-188)
// and of the manufactured flow used by its convergence tests
// (inc/manufactured.hpp:16-68).
#pragma once

#include <cmath>

#include "orc_assembly.hpp"

namespace orc {

// ------------------------------------------------------------ manufactured
namespace mms {
inline Real sqr(Real s) { return s * s; }
inline Real bump(Real s) { return sqr(s) * sqr(s - 1.0); }
inline Real bump_d1(Real s) { return 2.0 * s * (s - 1.0) * (2.0 * s - 1.0); }
inline Real bump_d2(Real s) { return 12.0 * s * s - 12.0 * s + 2.0; }
inline Real bump_d3(Real s) { return 24.0 * s - 12.0; }
/// divergence-free velocity vanishing on the unit-square boundary
inline V2 velocity(const V2& x) { return {-bump(x.x) * bump_d1(x.y), bump_d1(x.x) * bump(x.y)}; }
/// g[i][j] = d u_i / d x_j
inline void gradient(const V2& x, Real g[2][2]) {
  g[0][0] = -bump_d1(x.x) * bump_d1(x.y);
  g[0][1] = -bump(x.x) * bump_d2(x.y);
  g[1][0] = bump_d2(x.x) * bump(x.y);
  g[1][1] = bump_d1(x.x) * bump_d1(x.y);
}
inline V2 laplacian(const V2& x) {
  return {-bump_d2(x.x) * bump_d1(x.y) - bump(x.x) * bump_d3(x.y),
          bump_d3(x.x) * bump(x.y) + bump_d1(x.x) * bump_d2(x.y)};
}
inline Real pressure(const V2& x) { return x.x * (1.0 - x.x) * (1.0 - x.y) - 1.0 / 12.0; }
inline V2 pressure_gradient(const V2& x) { return {(1.0 - 2.0 * x.x) * (1.0 - x.y), x.x * x.x - x.x}; }
/// -nu lap u + beta u + grad p
inline V2 stokes_load(Real nu, Real beta, const V2& x) {
  const V2 l = laplacian(x), u = velocity(x), gp = pressure_gradient(x);
  return {-nu * l.x + beta * u.x + gp.x, -nu * l.y + beta * u.y + gp.y};
}
/// -nu lap u + (u . grad) u + grad p
inline V2 ns_load(Real nu, const V2& x) {
  const V2 l = laplacian(x), u = velocity(x), gp = pressure_gradient(x);
  Real g[2][2];
  gradient(x, g);
  return {-nu * l.x + g[0][0] * u.x + g[0][1] * u.y + gp.x, -nu * l.y + g[1][0] * u.x + g[1][1] * u.y + gp.y};
}
}  // namespace mms

/// The linear flow of the reference's exactness test (tests/test_postprocess.cpp:120-157).
namespace linflow {
inline V2 velocity(const V2& x) { return {1 + 2 * x.y + 3 * x.x, 4 - 3 * x.y + 5 * x.x}; }
inline void gradient(const V2&, Real g[2][2]) {
  g[0][0] = 3;
  g[0][1] = 2;
  g[1][0] = 5;
  g[1][1] = -3;
}
}  // namespace linflow

/// exact flows by kind: 1 manufactured, 2 linear
inline void exact_flow(int kind, const V2& x, V2& u, Real g[2][2]) {
  if (kind == 1) {
    u = mms::velocity(x);
    mms::gradient(x, g);
  } else {
    u = linflow::velocity(x);
    linflow::gradient(x, g);
  }
}

// ---------------------------------------------------------- post-processing
struct PostTables {
  int k = 0, ns = 1, ns_hi = 3;
  std::vector<Poly> hi;                       // orthonormal P^{k+1}
  std::vector<std::array<Poly, 2>> hi_grad;   // their reference gradients
  Real ref_mean = 0;                          // int_ref hi[0]
  TriRule err;                                // error rule (tri_rule(16), postprocess.hpp:113)
};

inline const PostTables& post_tables(int k) {
  static std::map<int, std::unique_ptr<PostTables>> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(k);
  if (it != cache.end()) return *it->second;
  auto t = std::make_unique<PostTables>();
  t->k = k;
  t->ns = int(orthonormal_basis(k).size());
  t->hi = orthonormal_basis(k + 1);
  t->ns_hi = int(t->hi.size());
  for (const Poly& p : t->hi) t->hi_grad.push_back({p.dx(), p.dy()});
  t->ref_mean = tri_l2(t->hi[0], Poly::mono(0, 0));
  t->err = tri_rule(16);
  auto [ins, ok] = cache.emplace(k, std::move(t));
  (void)ok;
  return *ins->second;
}

/// local RT coefficients of an HDG velocity on element e, orientation factors
/// applied (ElemCtx::val folds them into the tables instead)
inline Vec local_rt(const ElemCtx& cx, const Space& V, const Vec& compound, const Vec& interior, int e) {
  Vec c(cx.nrt);
  for (int le = 0; le < 3; ++le)
    for (int i = 0; i < cx.nfd; ++i) c[le * cx.nfd + i] = cx.geo.rt_factor(le, i) * compound[V.flux(cx.geo.facet[le], i)];
  for (int j = 0; j < cx.no; ++j) c[3 * cx.nfd + j] = interior[V.interior(e, j)];
  return c;
}

/// u* in [P^{k+1}]^2 per element: (grad u*, grad v) = -1/nu (L_h, grad v),
/// mean(u*) = mean(u_h); column-major [2 ns_hi] per element, x then y
/// (inc/postprocess.hpp:24-80). grad: [ne][4 ns] (recover_locals layout).
inline std::vector<Real> postprocess_velocity(const Mesh& mesh, const Space& V, Real nu, const Vec& compound,
                                              const Vec& interior, const std::vector<Real>& grad) {
  const PostTables& pt = post_tables(V.k);
  const RefData& rd = ref_data(V.k);
  const int ns = pt.ns, nh = pt.ns_hi, nq = rd.nq();
  std::vector<Real> out(std::size_t(mesh.ne()) * 2 * nh, 0.0);
  for (int e = 0; e < mesh.ne(); ++e) {
    ElemCtx cx(mesh, V, e);
    const Vec c = local_rt(cx, V, compound, interior, e);
    const Geo& g = cx.geo;
    Mat K(nh - 1, nh - 1), rhs(nh - 1, 2);
    Real um[2] = {0, 0};
    for (int q = 0; q < nq; ++q) {
      const Real w = rd.vol.wts[q];
      const V2 xh = rd.vol.pts[q];
      // physical gradients of the hi modes 1..nh-1: Ji^T grad_hat
      std::vector<Real> gx(nh), gy(nh);
      for (int s = 0; s < nh; ++s) {
        const Real a = pt.hi_grad[s][0].eval(xh.x, xh.y), b = pt.hi_grad[s][1].eval(xh.x, xh.y);
        gx[s] = g.Ji[0][0] * a + g.Ji[1][0] * b;
        gy[s] = g.Ji[0][1] * a + g.Ji[1][1] * b;
      }
      for (int s = 1; s < nh; ++s)
        for (int t = 1; t < nh; ++t) K(s - 1, t - 1) += w * g.detJ * (gx[s] * gx[t] + gy[s] * gy[t]);
      Real L[2][2];
      for (int comp = 0; comp < 4; ++comp) {
        Real v = 0;
        for (int m = 0; m < ns; ++m) v += rd.vscal(q, m) * grad[(std::size_t(e) * 4 + comp) * ns + m];
        L[comp / 2][comp % 2] = v;
      }
      for (int s = 1; s < nh; ++s)
        for (int i = 0; i < 2; ++i) rhs(s - 1, i) -= w * g.detJ / nu * (gx[s] * L[i][0] + gy[s] * L[i][1]);
      Real hx = 0, hy = 0;
      for (int r = 0; r < cx.nrt; ++r) {
        hx += rd.vval[q](0, r) * c[r];
        hy += rd.vval[q](1, r) * c[r];
      }
      const V2 v = g.applyJ(hx, hy) / g.detJ;  // reference weight: mean over the cell
      um[0] += w * v.x;
      um[1] += w * v.y;
    }
    LU lu(K);
    for (int comp = 0; comp < 2; ++comp) {
      Vec b(nh - 1);
      for (int s = 0; s < nh - 1; ++s) b[s] = rhs(s, comp);
      Vec x = lu.solve(b);
      out[std::size_t(e) * 2 * nh + comp * nh] = um[comp] / pt.ref_mean;
      for (int s = 0; s < nh - 1; ++s) out[std::size_t(e) * 2 * nh + comp * nh + 1 + s] = x[s];
    }
  }
  return out;
}

struct ErrorNorms {
  Real e_u = 0, e_L = 0, e_ustar = 0, div_u = 0;
};

/// inc/postprocess.hpp:142-188, against exact flow `kind`
inline ErrorNorms measure_errors(const Mesh& mesh, const Space& V, Real nu, const Vec& compound, const Vec& interior,
                                 const std::vector<Real>& grad, const std::vector<Real>& post, int kind) {
  const PostTables& pt = post_tables(V.k);
  const RefData& rd = ref_data(V.k);
  const int ns = pt.ns, nh = pt.ns_hi;
  const TriRule& R = pt.err;
  Real su = 0, sL = 0, sp = 0, sd = 0;
  for (int e = 0; e < mesh.ne(); ++e) {
    ElemCtx cx(mesh, V, e);
    const Vec c = local_rt(cx, V, compound, interior, e);
    const Geo& g = cx.geo;
    for (std::size_t q = 0; q < R.pts.size(); ++q) {
      const Real w = R.wts[q] * g.detJ;
      const V2 xh = R.pts[q], xq = g.map(xh);
      Real hx = 0, hy = 0, dv = 0;
      for (int r = 0; r < cx.nrt; ++r) {
        hx += rd.rt.val[r][0].eval(xh.x, xh.y) * c[r];
        hy += rd.rt.val[r][1].eval(xh.x, xh.y) * c[r];
        dv += rd.rt.div[r].eval(xh.x, xh.y) * c[r];
      }
      const V2 uh = g.applyJ(hx, hy) / g.detJ;
      V2 ue;
      Real ge[2][2];
      exact_flow(kind, xq, ue, ge);
      su += w * ((ue.x - uh.x) * (ue.x - uh.x) + (ue.y - uh.y) * (ue.y - uh.y));
      sd += w * (dv / g.detJ) * (dv / g.detJ);
      for (int comp = 0; comp < 4; ++comp) {
        Real Lh = 0;
        for (int m = 0; m < ns; ++m)
          Lh += rd.scalar[m].eval(xh.x, xh.y) * grad[(std::size_t(e) * 4 + comp) * ns + m];
        const Real d = -nu * ge[comp / 2][comp % 2] - Lh;
        sL += w * d * d;
      }
      Real usx = 0, usy = 0;
      for (int s = 0; s < nh; ++s) {
        const Real p = pt.hi[s].eval(xh.x, xh.y);
        usx += p * post[std::size_t(e) * 2 * nh + s];
        usy += p * post[std::size_t(e) * 2 * nh + nh + s];
      }
      sp += w * ((ue.x - usx) * (ue.x - usx) + (ue.y - usy) * (ue.y - usy));
    }
  }
  return {std::sqrt(su), std::sqrt(sL), std::sqrt(sp), std::sqrt(sd)};
}

}  // namespace orc
