// TEST INFRASTRUCTURE ONLY (see orc_core.hpp). Sparse matrices, element
// local blocks, static condensation, condensed assembly, divergence rows,
// grad-div penalty and local recovery (reference inc/assembly.hpp).
#pragma once

#include "orc_fe.hpp"

namespace orc {

// --------------------------------------------------------------- sparse ----
struct Trip {
  Index i, j;
  Real v;
};

/// Compressed sparse row matrix, sorted columns, duplicates summed in
/// insertion order (role of Eigen setFromTriplets).
struct Csr {
  Index rows = 0, cols = 0;
  std::vector<Index> ptr{0};
  std::vector<Index> idx;
  std::vector<Real> val;

  static Csr from_trips(Index r, Index c, const std::vector<Trip>& t, bool prune_zero = false) {
    Csr m;
    m.rows = r;
    m.cols = c;
    std::vector<Index> cnt(r + 1, 0);
    for (const auto& x : t) cnt[x.i + 1]++;
    for (Index i = 0; i < r; ++i) cnt[i + 1] += cnt[i];
    std::vector<Index> cj(t.size());
    std::vector<Real> cv(t.size());
    std::vector<Index> pos(cnt.begin(), cnt.end() - 1);
    for (const auto& x : t) {  // stable bucket by row keeps insertion order
      cj[pos[x.i]] = x.j;
      cv[pos[x.i]] = x.v;
      pos[x.i]++;
    }
    m.ptr.assign(r + 1, 0);
    std::vector<Index> ord;
    for (Index i = 0; i < r; ++i) {
      Index b = cnt[i], e = cnt[i + 1];
      ord.resize(e - b);
      std::iota(ord.begin(), ord.end(), b);
      std::stable_sort(ord.begin(), ord.end(), [&](Index p, Index q) { return cj[p] < cj[q]; });
      Index last = -1;
      for (Index p : ord) {
        if (cj[p] == last) {
          m.val.back() += cv[p];
        } else {
          m.idx.push_back(cj[p]);
          m.val.push_back(cv[p]);
          last = cj[p];
        }
      }
      if (prune_zero) {
        Index keep = m.ptr[i];
        for (Index p = m.ptr[i]; p < Index(m.idx.size()); ++p)
          if (m.val[p] != 0.0) {
            m.idx[keep] = m.idx[p];
            m.val[keep] = m.val[p];
            ++keep;
          }
        m.idx.resize(keep);
        m.val.resize(keep);
      }
      m.ptr[i + 1] = Index(m.idx.size());
    }
    return m;
  }
  Index nnz() const { return Index(val.size()); }
  Real coeff(Index i, Index j) const {
    auto b = idx.begin() + ptr[i], e = idx.begin() + ptr[i + 1];
    auto it = std::lower_bound(b, e, j);
    return (it != e && *it == j) ? val[it - idx.begin()] : 0.0;
  }
  Vec mul(const Vec& x) const {
    Vec y(rows, 0.0);
    for (Index i = 0; i < rows; ++i) {
      Real s = 0;
      for (Index p = ptr[i]; p < ptr[i + 1]; ++p) s += val[p] * x[idx[p]];
      y[i] = s;
    }
    return y;
  }
  Csr transpose() const {
    std::vector<Trip> t;
    t.reserve(val.size());
    for (Index i = 0; i < rows; ++i)
      for (Index p = ptr[i]; p < ptr[i + 1]; ++p) t.push_back({idx[p], i, val[p]});
    return from_trips(cols, rows, t);
  }
  /// this + s * B (same shape)
  Csr add(const Csr& B, Real s) const {
    std::vector<Trip> t;
    t.reserve(val.size() + B.val.size());
    for (Index i = 0; i < rows; ++i) {
      for (Index p = ptr[i]; p < ptr[i + 1]; ++p) t.push_back({i, idx[p], val[p]});
      for (Index p = B.ptr[i]; p < B.ptr[i + 1]; ++p) t.push_back({i, B.idx[p], s * B.val[p]});
    }
    return from_trips(rows, cols, t);
  }
  Mat dense() const {
    Mat D{static_cast<int>(rows), static_cast<int>(cols)};
    for (Index i = 0; i < rows; ++i)
      for (Index p = ptr[i]; p < ptr[i + 1]; ++p) D(int(i), int(idx[p])) = val[p];
    return D;
  }
};

inline Csr spmul(const Csr& A, const Csr& B) {
  std::vector<Trip> t;
  for (Index i = 0; i < A.rows; ++i)
    for (Index p = A.ptr[i]; p < A.ptr[i + 1]; ++p) {
      Index k = A.idx[p];
      for (Index q = B.ptr[k]; q < B.ptr[k + 1]; ++q) t.push_back({i, B.idx[q], A.val[p] * B.val[q]});
    }
  return Csr::from_trips(A.rows, B.cols, t);
}

// ------------------------------------------------------------- assembly ----
struct AsmOpt {
  Real nu = 1.0, beta = 0.0, mass_coef = 0.0;
  Field load;
  std::function<V2(int elem, const V2& x)> elem_load;  // optional element-aware load
  const HDGVel* advection = nullptr;
  bool newton = false;
  const HDGVel* mass_field = nullptr;
};

/// Per-element tables with orientation factors applied; local order:
/// 3(k+1) flux, 3(k+1) tangential, k(k+1) interior (inc/assembly.hpp:84-189).
struct ElemCtx {
  const RefData* rd;
  Geo geo;
  int k, nfd, nc, nrt, no, nv, ns;
  std::vector<Index> gdof;
  std::vector<Mat> val, jac;  // per q: 2 x nrt, 4 x nrt
  Mat div;                    // nq x nrt
  std::array<std::vector<Mat>, 3> trace, tdiff;  // per edge per point: 2 x nv
  std::array<V2, 3> n_out;
  std::array<Real, 3> ds;
  int vel_of_rt(int r) const { return r < 3 * nfd ? r : nc + (r - 3 * nfd); }

  ElemCtx(const Mesh& mesh, const Space& V, int e) : rd(&ref_data(V.k)), geo(mesh, e) {
    k = V.k;
    nfd = k + 1;
    nc = 6 * nfd;
    no = V.n_int();
    nrt = 3 * nfd + no;
    nv = nc + no;
    ns = rd->ns();
    gdof.resize(nc);
    for (int le = 0; le < 3; ++le)
      for (int i = 0; i < nfd; ++i) {
        gdof[le * nfd + i] = V.flux(geo.facet[le], i);
        gdof[3 * nfd + le * nfd + i] = V.tang(geo.facet[le], i);
      }
    Vec factor(nrt, 1.0);
    for (int le = 0; le < 3; ++le)
      for (int i = 0; i < nfd; ++i) factor[le * nfd + i] = geo.rt_factor(le, i);
    const int nq = rd->nq();
    val.assign(nq, Mat(2, nrt));
    jac.assign(nq, Mat(4, nrt));
    div = Mat(nq, nrt);
    const Real (&J)[2][2] = geo.J;
    const Real (&Ji)[2][2] = geo.Ji;
    for (int q = 0; q < nq; ++q) {
      for (int a = 0; a < nrt; ++a) {
        V2 v = geo.applyJ(rd->vval[q](0, a), rd->vval[q](1, a)) / geo.detJ;
        val[q](0, a) = v.x * factor[a];
        val[q](1, a) = v.y * factor[a];
        Real Jh[2][2] = {{rd->vjac[q](0, a), rd->vjac[q](1, a)}, {rd->vjac[q](2, a), rd->vjac[q](3, a)}};
        Real T[2][2], P[2][2];
        for (int i = 0; i < 2; ++i)
          for (int j = 0; j < 2; ++j) T[i][j] = J[i][0] * Jh[0][j] + J[i][1] * Jh[1][j];
        for (int i = 0; i < 2; ++i)
          for (int j = 0; j < 2; ++j) P[i][j] = (T[i][0] * Ji[0][j] + T[i][1] * Ji[1][j]) / geo.detJ;
        jac[q](0, a) = P[0][0] * factor[a];
        jac[q](1, a) = P[0][1] * factor[a];
        jac[q](2, a) = P[1][0] * factor[a];
        jac[q](3, a) = P[1][1] * factor[a];
        div(q, a) = rd->vdiv(q, a) / geo.detJ * factor[a];
      }
    }
    const int nqe = rd->nqe();
    for (int le = 0; le < 3; ++le) {
      V2 tf = mesh.ftan(geo.facet[le]);
      V2 n = mesh.fnormal(geo.facet[le]) * Real(geo.sigma[le]);
      n_out[le] = n;
      ds[le] = 0.5 * geo.flen[le];
      trace[le].assign(nqe, Mat(2, nv));
      tdiff[le].assign(nqe, Mat(2, nv));
      for (int q = 0; q < nqe; ++q) {
        Mat& T = trace[le][q];
        Mat& D = tdiff[le][q];
        for (int a = 0; a < nrt; ++a) {
          int col = vel_of_rt(a);
          V2 ph = geo.applyJ(rd->eval_[le][q](0, a), rd->eval_[le][q](1, a)) / geo.detJ;
          T(0, col) = factor[a] * ph.x;
          T(1, col) = factor[a] * ph.y;
          Real tn = T(0, col) * n.x + T(1, col) * n.y;
          D(0, col) = T(0, col) - tn * n.x;
          D(1, col) = T(1, col) - tn * n.y;
        }
        Real t = rd->edge.pts[q];
        for (int i = 0; i < nfd; ++i) {
          Real lg = legendre(i, t);
          if (geo.rho[le] < 0 && i % 2 == 1) lg = -lg;
          int col = 3 * nfd + le * nfd + i;
          T(0, col) = lg * tf.x;
          T(1, col) = lg * tf.y;
          D(0, col) = -T(0, col);
          D(1, col) = -T(1, col);
        }
      }
    }
  }
  Vec local_velocity(const HDGVel& u, int e) const {
    Vec x(nv);
    for (int a = 0; a < nc; ++a) x[a] = u.compound[gdof[a]];
    for (int j = 0; j < no; ++j) x[nc + j] = u.interior[u.V.interior(e, j)];
    return x;
  }
  Vec rt_coeffs(const Vec& xl) const {
    Vec c(nrt);
    for (int a = 0; a < 3 * nfd; ++a) c[a] = xl[a];
    for (int j = 0; j < no; ++j) c[3 * nfd + j] = xl[nc + j];
    return c;
  }
};

struct LocalBlocks {
  Mat A, P, C;
  Vec rhs;
};

/// Element matrices before condensation (inc/assembly.hpp:205-336).
inline LocalBlocks local_blocks(const ElemCtx& cx, int e, const AsmOpt& opt) {
  const RefData& rd = *cx.rd;
  const int nv = cx.nv, nrt = cx.nrt, ns = cx.ns, nfd = cx.nfd;
  LocalBlocks b;
  b.C = Mat(4 * ns, nv);
  b.A = Mat(nv, nv);
  b.P = Mat(ns - 1, nv);
  b.rhs.assign(nv, 0.0);
  Vec xw, wrt, mrt;
  if (opt.advection) {
    xw = cx.local_velocity(*opt.advection, e);
    wrt = cx.rt_coeffs(xw);
  }
  if (opt.mass_field) mrt = cx.rt_coeffs(cx.local_velocity(*opt.mass_field, e));
  const Real mass = opt.beta + opt.mass_coef;
  for (int q = 0; q < rd.nq(); ++q) {
    const Real w = rd.vol.wts[q] * cx.geo.detJ;
    const Mat& V = cx.val[q];
    const Mat& J = cx.jac[q];
    for (int r = 0; r < nrt; ++r) {
      int a = cx.vel_of_rt(r);
      for (int c = 0; c < 4; ++c)
        for (int m = 0; m < ns; ++m) b.C(c * ns + m, a) += w * J(c, r) * rd.vscal(q, m);
      for (int m = 1; m < ns; ++m) b.P(m - 1, a) += w * cx.div(q, r) * rd.vscal(q, m);
    }
    if (mass != 0.0)
      for (int r = 0; r < nrt; ++r)
        for (int s = 0; s < nrt; ++s)
          b.A(cx.vel_of_rt(r), cx.vel_of_rt(s)) += mass * w * (V(0, r) * V(0, s) + V(1, r) * V(1, s));
    if (opt.load || opt.elem_load || opt.mass_field) {
      V2 fv;
      V2 xq = cx.geo.map(rd.vol.pts[q]);
      if (opt.elem_load) fv = opt.elem_load(e, xq);
      else if (opt.load) fv = opt.load(xq);
      if (opt.mass_field) {
        Real sx = 0, sy = 0;
        for (int r = 0; r < nrt; ++r) { sx += V(0, r) * mrt[r]; sy += V(1, r) * mrt[r]; }
        fv += V2(sx, sy) * opt.mass_coef;
      }
      for (int r = 0; r < nrt; ++r) b.rhs[cx.vel_of_rt(r)] += w * (fv.x * V(0, r) + fv.y * V(1, r));
    }
    if (opt.advection) {
      Real wx = 0, wy = 0;
      for (int r = 0; r < nrt; ++r) { wx += V(0, r) * wrt[r]; wy += V(1, r) * wrt[r]; }
      for (int r = 0; r < nrt; ++r) {
        int a = cx.vel_of_rt(r);
        Real g[4] = {J(0, r), J(1, r), J(2, r), J(3, r)};
        for (int s = 0; s < nrt; ++s) {
          int bb = cx.vel_of_rt(s);
          Real t = V(0, s) * (g[0] * wx + g[1] * wy) + V(1, s) * (g[2] * wx + g[3] * wy);
          b.A(a, bb) -= w * t;
          if (opt.newton) {
            Real tn = wx * (g[0] * V(0, s) + g[1] * V(1, s)) + wy * (g[2] * V(0, s) + g[3] * V(1, s));
            b.A(a, bb) -= w * tn;
          }
        }
        if (opt.newton) b.rhs[a] -= w * (wx * (g[0] * wx + g[1] * wy) + wy * (g[2] * wx + g[3] * wy));
      }
    }
  }
  for (int le = 0; le < 3; ++le) {
    const V2 n = cx.n_out[le];
    for (int q = 0; q < rd.nqe(); ++q) {
      const Real wds = rd.edge.wts[q] * cx.ds[le];
      const Mat& T = cx.trace[le][q];
      const Mat& D = cx.tdiff[le][q];
      const Real nn[2] = {n.x, n.y};
      for (int a = 0; a < nv; ++a) {
        if (D(0, a) == 0.0 && D(1, a) == 0.0) continue;
        for (int i = 0; i < 2; ++i)
          for (int j = 0; j < 2; ++j)
            for (int m = 0; m < ns; ++m) b.C((i * 2 + j) * ns + m, a) -= wds * D(i, a) * nn[j] * rd.escal[le](q, m);
      }
      if (opt.advection) {
        Real wtx = 0, wty = 0;
        for (int a = 0; a < 3 * nfd; ++a) { wtx += T(0, a) * xw[a]; wty += T(1, a) * xw[a]; }
        for (int j = 0; j < cx.no; ++j) { wtx += T(0, cx.nc + j) * xw[cx.nc + j]; wty += T(1, cx.nc + j) * xw[cx.nc + j]; }
        Real wn = wtx * n.x + wty * n.y;
        V2 tsk;  // tangential skeleton trace of the wind on this edge
        for (int a = 3 * nfd; a < 6 * nfd; ++a) { tsk.x += T(0, a) * xw[a]; tsk.y += T(1, a) * xw[a]; }
        // round-off guard: |w.n| below 1e-13 of the magnitude of the terms it
        // is summed from (|RT coefficient| x |basis trace|, plus the
        // tangential skeleton trace) is the exact-arithmetic w.n = 0 (inflow
        // branch), not a basis-dependent round-off sign (no-slip walls, the lid,
        // a solenoidal wind along the boundary, nodes where the wind vanishes)
        Real wabs = std::sqrt(tsk.x * tsk.x + tsk.y * tsk.y);
        for (int a = 0; a < 3 * nfd; ++a) wabs += std::abs(xw[a]) * std::sqrt(T(0, a) * T(0, a) + T(1, a) * T(1, a));
        for (int j = 0; j < cx.no; ++j)
          wabs += std::abs(xw[cx.nc + j]) * std::sqrt(T(0, cx.nc + j) * T(0, cx.nc + j) + T(1, cx.nc + j) * T(1, cx.nc + j));
        if (std::abs(wn) <= 1e-13 * wabs) wn = 0.0;
        const bool outflow = wn > 0;
        const V2 up0 = outflow ? V2(wtx, wty) : tsk;
        for (int a = 0; a < nv; ++a) {
          V2 ta(D(0, a), D(1, a));
          if (ta.x == 0.0 && ta.y == 0.0) continue;
          if (wn != 0.0) {
            if (outflow) {
              for (int r = 0; r < nrt; ++r) {
                int bb = cx.vel_of_rt(r);
                b.A(a, bb) += wds * wn * (ta.x * T(0, bb) + ta.y * T(1, bb));
              }
            } else {
              for (int i = 0; i < nfd * 3; ++i) {
                int bb = 3 * nfd + i;
                b.A(a, bb) += wds * wn * (ta.x * T(0, bb) + ta.y * T(1, bb));
              }
            }
          }
          if (opt.newton) {
            Real tup = ta.dot(up0);
            if (tup != 0.0)
              for (int i = 0; i < 3 * nfd; ++i) b.A(a, i) += wds * tup * (T(0, i) * n.x + T(1, i) * n.y);
            b.rhs[a] += wds * wn * tup;
          }
        }
      }
    }
  }
  // A += (nu/detJ) C^T C
  const Real s = opt.nu / cx.geo.detJ;
  for (int a = 0; a < nv; ++a)
    for (int c = 0; c < nv; ++c) {
      Real acc = 0;
      for (int r = 0; r < 4 * ns; ++r) acc += b.C(r, a) * b.C(r, c);
      b.A(a, c) += s * acc;
    }
  return b;
}

/// Schur complement of interior velocity and zero-mean pressure modes
/// (inc/assembly.hpp:341-364).
inline void condense(const ElemCtx& cx, const LocalBlocks& b, Mat& Ac, Vec& rc) {
  const int nc = cx.nc, no = cx.no, np = cx.ns - 1;
  if (no + np == 0) {
    Ac = b.A;
    rc = b.rhs;
    return;
  }
  const int nz = no + np;
  Mat Mzz(nz, nz), Mzc(nz, nc), Mcz(nc, nz);
  for (int i = 0; i < no; ++i)
    for (int j = 0; j < no; ++j) Mzz(i, j) = b.A(nc + i, nc + j);
  for (int i = 0; i < no; ++i)
    for (int m = 0; m < np; ++m) {
      Mzz(i, no + m) = -b.P(m, nc + i);
      Mzz(no + m, i) = -b.P(m, nc + i);
    }
  for (int j = 0; j < nc; ++j) {
    for (int i = 0; i < no; ++i) Mzc(i, j) = b.A(nc + i, j);
    for (int m = 0; m < np; ++m) Mzc(no + m, j) = -b.P(m, j);
    for (int i = 0; i < no; ++i) Mcz(j, i) = b.A(j, nc + i);
    for (int m = 0; m < np; ++m) Mcz(j, no + m) = -b.P(m, j);
  }
  LU lu(Mzz);
  Mat X = lu.solve(Mzc);
  Mat MX = matmul(Mcz, X);
  Ac = Mat(nc, nc);
  for (int i = 0; i < nc; ++i)
    for (int j = 0; j < nc; ++j) Ac(i, j) = b.A(i, j) - MX(i, j);
  Vec rz(nz, 0.0);
  for (int i = 0; i < no; ++i) rz[i] = b.rhs[nc + i];
  Vec y = lu.solve(rz);
  Vec my = matvec(Mcz, y);
  rc.assign(nc, 0.0);
  for (int i = 0; i < nc; ++i) rc[i] = b.rhs[i] - my[i];
}

struct Condensed {
  Csr A;
  Vec rhs;
};

/// (inc/assembly.hpp:374-406)
inline Condensed assemble_condensed(const Mesh& mesh, const Space& V, const Constraints& con, const AsmOpt& opt) {
  Condensed s;
  s.rhs.assign(con.n_free, 0.0);
  std::vector<Trip> t;
  t.reserve(std::size_t(mesh.ne()) * 36 * (V.k + 1) * (V.k + 1));
  Mat Ac;
  Vec rc;
  for (int e = 0; e < mesh.ne(); ++e) {
    ElemCtx cx(mesh, V, e);
    LocalBlocks b = local_blocks(cx, e, opt);
    condense(cx, b, Ac, rc);
    for (int a = 0; a < cx.nc; ++a) {
      Index fa = con.full_to_free[cx.gdof[a]];
      if (fa < 0) continue;
      s.rhs[fa] += rc[a];
      for (int c = 0; c < cx.nc; ++c) {
        Index fb = con.full_to_free[cx.gdof[c]];
        if (fb >= 0) t.push_back({fa, fb, Ac(a, c)});
        else s.rhs[fa] -= Ac(a, c) * con.g_full[cx.gdof[c]];
      }
    }
  }
  s.A = Csr::from_trips(con.n_free, con.n_free, t);
  return s;
}

/// Boundary-flux rows sigma|F| (inc/assembly.hpp:410-424); ne x n_compound.
inline Csr divergence_rows(const Space& V) {
  const Mesh& m = *V.mesh;
  std::vector<Trip> t;
  for (int e = 0; e < m.ne(); ++e)
    for (int le = 0; le < 3; ++le)
      t.push_back({e, V.flux(m.el[e].facet[le], 0), Real(m.el[e].sigma[le]) * m.flen(m.el[e].facet[le])});
  return Csr::from_trips(m.ne(), V.n_compound(), t);
}

inline Vec element_areas(const Mesh& m) {
  Vec a(m.ne());
  for (int e = 0; e < m.ne(); ++e) a[e] = m.area(e);
  return a;
}

/// D = sum_K |K|^-1 b_K b_K^T on free DOFs (inc/assembly.hpp:435-464).
inline Csr grad_div(const Space& V, const Constraints& con, const Vec& g_full, Vec* rhs) {
  const Mesh& m = *V.mesh;
  if (rhs) rhs->assign(con.n_free, 0.0);
  std::vector<Trip> t;
  for (int e = 0; e < m.ne(); ++e) {
    const auto& E = m.el[e];
    const Real ia = 1.0 / m.area(e);
    for (int i = 0; i < 3; ++i) {
      Index gi = V.flux(E.facet[i], 0), fi = con.full_to_free[gi];
      if (fi < 0) continue;
      Real bi = Real(E.sigma[i]) * m.flen(E.facet[i]);
      for (int j = 0; j < 3; ++j) {
        Index gj = V.flux(E.facet[j], 0), fj = con.full_to_free[gj];
        Real bj = Real(E.sigma[j]) * m.flen(E.facet[j]);
        if (fj >= 0) t.push_back({fi, fj, ia * bi * bj});
        else if (rhs) (*rhs)[fi] -= ia * bi * bj * g_full[gj];
      }
    }
  }
  return Csr::from_trips(con.n_free, con.n_free, t);
}

struct LocalSolution {
  Vec interior, p_ortho;
  Mat grad;  // 4 ns x ne
};

/// Re-eliminated locals from a skeleton solution (inc/assembly.hpp:513-549).
inline LocalSolution recover_locals(const Mesh& mesh, const Space& V, const AsmOpt& opt, const Vec& compound_full) {
  const int ns = ref_data(V.k).ns(), no = V.n_int(), np = ns - 1;
  LocalSolution out;
  out.interior.assign(V.n_interior(), 0.0);
  out.p_ortho.assign(std::size_t(mesh.ne()) * np, 0.0);
  out.grad = Mat(4 * ns, mesh.ne());
  for (int e = 0; e < mesh.ne(); ++e) {
    ElemCtx cx(mesh, V, e);
    LocalBlocks b = local_blocks(cx, e, opt);
    Vec xc(cx.nc), xv(cx.nv, 0.0);
    for (int a = 0; a < cx.nc; ++a) xv[a] = xc[a] = compound_full[cx.gdof[a]];
    if (no + np > 0) {
      const int nz = no + np;
      Mat Mzz(nz, nz), Mzc(nz, cx.nc);
      for (int i = 0; i < no; ++i)
        for (int j = 0; j < no; ++j) Mzz(i, j) = b.A(cx.nc + i, cx.nc + j);
      for (int i = 0; i < no; ++i)
        for (int m = 0; m < np; ++m) {
          Mzz(i, no + m) = -b.P(m, cx.nc + i);
          Mzz(no + m, i) = -b.P(m, cx.nc + i);
        }
      for (int j = 0; j < cx.nc; ++j) {
        for (int i = 0; i < no; ++i) Mzc(i, j) = b.A(cx.nc + i, j);
        for (int m = 0; m < np; ++m) Mzc(no + m, j) = -b.P(m, j);
      }
      Vec rz(nz, 0.0);
      for (int i = 0; i < no; ++i) rz[i] = b.rhs[cx.nc + i];
      Vec mx = matvec(Mzc, xc);
      for (int i = 0; i < nz; ++i) rz[i] -= mx[i];
      Vec z = LU(Mzz).solve(rz);
      for (int j = 0; j < no; ++j) out.interior[V.interior(e, j)] = z[j];
      for (int m = 0; m < np; ++m) out.p_ortho[std::size_t(e) * np + m] = z[no + m];
      for (int j = 0; j < no; ++j) xv[cx.nc + j] = z[j];
    }
    Vec cxv = matvec(b.C, xv);
    for (int r = 0; r < 4 * ns; ++r) out.grad(r, e) = -(opt.nu / cx.geo.detJ) * cxv[r];
  }
  return out;
}

}  // namespace orc
