// Advection (Oseen) state on the host: interpolation of a wind field into
// the hybrid RT_k space (reference inc/assembly.hpp:40-62 interpolate_hdg,
// inc/fespace.hpp:404-461 interpolate_rt) in THIS library's interior basis,
// its lowest-order carrier (inc/transfer.hpp:186-195) and the restriction
// down the mesh hierarchy (inc/transfer.hpp:164-182). Setup only.
#pragma once

#include <functional>
#include <vector>

#include "basis.hpp"
#include "plan.hpp"
#include "transfer.hpp"

namespace hpmg {
namespace host {

using PointField = std::function<void(double x, double y, double* out)>;

struct HdgField {
  int k = 0;
  std::vector<double> compound;  // reference layout: all flux (f*nfd+i), then all tangential
  std::vector<double> interior;  // [ne][k(k+1)]
};

inline HdgField interpolate_hdg(const TriMesh& m, int k, const RefTensors& T, const PointField& field) {
  HdgField u;
  u.k = k;
  const int nfd = k + 1, no = T.no, nrt = T.nrt;
  const int64_t nflux = int64_t(m.nf()) * nfd;
  u.compound.assign(2 * nflux, 0.0);
  u.interior.assign(size_t(m.ne()) * no, 0.0);
  std::vector<double> ex, ew;
  gauss(3 * k + 4, ex, ew);
  double L[8], v[2];
  for (int f = 0; f < m.nf(); ++f) {
    double nx, ny, tx, ty;
    m.fnormal(f, nx, ny);
    m.ftan(f, tx, ty);
    for (size_t q = 0; q < ex.size(); ++q) {
      double x, y;
      m.fpoint(f, ex[q], x, y);
      field(x, y, v);
      legendre(k, ex[q], L);
      const double vn = v[0] * nx + v[1] * ny, vt = v[0] * tx + v[1] * ty;
      for (int i = 0; i <= k; ++i) {
        const double w = 0.5 * (2 * i + 1) * ew[q] * L[i];
        u.compound[size_t(f) * nfd + i] += w * vn;
        u.compound[nflux + size_t(f) * nfd + i] += w * vt;
      }
    }
  }
  if (no == 0) return u;
  std::vector<double> A(size_t(no) * no), b(no);
  for (int e = 0; e < m.ne(); ++e) {
    const ElemGeo g = element_geometry(m, e);
    std::fill(A.begin(), A.end(), 0.0);
    std::fill(b.begin(), b.end(), 0.0);
    const double x0 = m.vx[m.ev[e][0]], y0 = m.vy[m.ev[e][0]];
    for (int q = 0; q < T.nq; ++q) {
      const double w = T.qw[q] * g.detJ;
      auto phys = [&](int r, double& px, double& py) {
        const double a0 = T.vval[(size_t(q) * 2) * nrt + r], a1 = T.vval[(size_t(q) * 2 + 1) * nrt + r];
        px = (g.J[0] * a0 + g.J[1] * a1) / g.detJ;
        py = (g.J[2] * a0 + g.J[3] * a1) / g.detJ;
      };
      field(x0 + g.J[0] * T.qx[q] + g.J[1] * T.qy[q], y0 + g.J[2] * T.qx[q] + g.J[3] * T.qy[q], v);
      double gx = v[0], gy = v[1];
      for (int le = 0; le < 3; ++le)
        for (int i = 0; i <= k; ++i) {
          double f = g.fac[le];
          if ((i & 1) && g.rho[le] < 0) f = -f;
          const double c = u.compound[size_t(m.ef[e][le]) * nfd + i] * f;
          double px, py;
          phys(le * nfd + i, px, py);
          gx -= c * px;
          gy -= c * py;
        }
      for (int a = 0; a < no; ++a) {
        double ax, ay;
        phys(3 * nfd + a, ax, ay);
        b[a] += w * (ax * gx + ay * gy);
        for (int c = 0; c < no; ++c) {
          double cx, cy;
          phys(3 * nfd + c, cx, cy);
          A[size_t(a) * no + c] += w * (ax * cx + ay * cy);
        }
      }
    }
    std::vector<double> sol = b;
    lu_solve_multi(A, no, sol, 1);
    for (int j = 0; j < no; ++j) u.interior[size_t(e) * no + j] = sol[j];
  }
  return u;
}

/// Lowest-order carrier on the same mesh: constant facet modes only.
inline HdgField lowest_order(const TriMesh& m, const HdgField& wk) {
  HdgField w0;
  const int nfd = wk.k + 1;
  const int64_t nf = m.nf(), nflux = nf * nfd;
  w0.compound.assign(2 * nf, 0.0);
  for (int64_t f = 0; f < nf; ++f) {
    w0.compound[f] = wk.compound[f * nfd];
    w0.compound[nf + f] = wk.compound[nflux + f * nfd];
  }
  return w0;
}

/// Coarse carrier: average of the two children, reoriented (transfer.hpp:164-182).
inline HdgField restrict_wind(const TriMesh& cm, const TriMesh& fm, const Refinement& R, const HdgField& wf) {
  HdgField wc;
  const int64_t ncf = cm.nf(), nff = fm.nf();
  wc.compound.assign(2 * ncf, 0.0);
  for (int cf = 0; cf < cm.nf(); ++cf) {
    double nx, ny;
    cm.fnormal(cf, nx, ny);
    double flux = 0, tang = 0;
    for (int c = 0; c < 2; ++c) {
      const int ff = R.fchildren[cf][c];
      double fx, fy;
      fm.fnormal(ff, fx, fy);
      const double s = (nx * fx + ny * fy) > 0 ? 0.5 : -0.5;
      flux += s * wf.compound[ff];
      tang += s * wf.compound[nff + ff];
    }
    wc.compound[cf] = flux;
    wc.compound[ncf + cf] = tang;
  }
  return wc;
}

/// Per-element local wind coefficients in the condensation's local order
/// (3 nfd flux, 3 nfd tangential, then interior).
inline std::vector<double> local_wind(const TriMesh& m, int k, const HdgField& w) {
  const int nfd = k + 1, nc = 6 * nfd, no = k * (k + 1), nv = nc + no;
  const int64_t nflux = int64_t(m.nf()) * nfd;
  std::vector<double> x(size_t(m.ne()) * nv, 0.0);
  for (int e = 0; e < m.ne(); ++e) {
    double* xe = &x[size_t(e) * nv];
    for (int le = 0; le < 3; ++le)
      for (int i = 0; i < nfd; ++i) {
        const int64_t f = m.ef[e][le];
        xe[le * nfd + i] = w.compound[f * nfd + i];
        xe[3 * nfd + le * nfd + i] = w.compound[nflux + f * nfd + i];
      }
    for (int j = 0; j < no; ++j) xe[nc + j] = w.interior[size_t(e) * no + j];
  }
  return x;
}

}  // namespace host
}  // namespace hpmg
