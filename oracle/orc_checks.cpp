// TEST INFRASTRUCTURE ONLY (see orc_core.hpp). Restatements of the
// reference's element-level known-answer tests; each returns the measured
// quantities and tests/test_oracle_pins.py applies the reference thresholds.
#include <random>

#include "orc_mg.hpp"
#include "orc_post.hpp"

using namespace orc;

namespace {
Mesh retag_outflow(Mesh m) {
  for (auto& f : m.fc)
    if (f.tag == kDirichlet) f.tag = kOutflow;
  return m;
}
Real frob(const Mat& A) {
  Real s = 0;
  for (Real v : A.a) s += v * v;
  return std::sqrt(s);
}
bool cholesky_ok(const Mat& A) {
  int n = A.r;
  Mat L(n, n);
  for (int j = 0; j < n; ++j) {
    Real d = A(j, j);
    for (int k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
    if (!(d > 0)) return false;
    L(j, j) = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      Real s = A(i, j);
      for (int k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
      L(i, j) = s / L(j, j);
    }
  }
  return true;
}
}  // namespace

extern "C" {

/// test_fespace.cpp:27-100: dims, facet traces = L_i, higher facet functions
/// divergence-free, interior functions have zero normal trace.
/// out: [dim ok, max trace err, max div err, max interior trace err]
void orc_check_rt(int k, double* out) {
  const RTRef& rt = ref_data(k).rt;
  out[0] = (rt.dim == (k + 1) * (k + 3) && rt.n_bubble == k * (k - 1) / 2 &&
            rt.n_div == (k + 1) * (k + 2) / 2 - 1)
               ? 1.0
               : 0.0;
  const auto& E = ref_edges();
  LineRule lr = line_rule(12);
  Real tr = 0, dv = 0, it = 0;
  for (int e = 0; e < 3; ++e)
    for (int i = 0; i <= k; ++i) {
      int fn = rt.facet_fn(e, i);
      for (int g = 0; g < 3; ++g)
        for (std::size_t q = 0; q < lr.pts.size(); ++q) {
          Real t = lr.pts[q];
          V2 x = (E[g].a * (1 - t) + E[g].b * (1 + t)) * 0.5;
          Real vn = rt.val[fn][0].eval(x.x, x.y) * E[g].n_out.x + rt.val[fn][1].eval(x.x, x.y) * E[g].n_out.y;
          tr = std::max(tr, std::abs(vn - (g == e ? legendre(i, t) : 0.0)));
        }
      if (i >= 1)
        for (int q = 0; q < 8; ++q) dv = std::max(dv, std::abs(rt.div[fn].eval(0.3, 0.2 + 0.04 * q)));
    }
  for (int j = 0; j < rt.n_interior(); ++j)
    for (int g = 0; g < 3; ++g)
      for (std::size_t q = 0; q < lr.pts.size(); ++q) {
        Real t = lr.pts[q];
        V2 x = (E[g].a * (1 - t) + E[g].b * (1 + t)) * 0.5;
        int fn = rt.interior_fn(j);
        Real vn = rt.val[fn][0].eval(x.x, x.y) * E[g].n_out.x + rt.val[fn][1].eval(x.x, x.y) * E[g].n_out.y;
        it = std::max(it, std::abs(vn));
      }
  out[1] = tr;
  out[2] = dv;
  out[3] = it;
}

/// test_assembly.cpp:24-38: condensed operator symmetric and SPD.
/// out: [relative asymmetry, spd(1/0)]
void orc_check_condensed_spd(int k, double* out) {
  Mesh mesh = unit_square(2);
  Space V(mesh, k);
  Constraints con = Constraints::build(V, nullptr);
  AsmOpt opt;
  opt.nu = 1.7;
  opt.beta = 0.4;
  Mat A = assemble_condensed(mesh, V, con, opt).A.dense();
  Mat D = A;
  for (int i = 0; i < A.r; ++i)
    for (int j = 0; j < A.c; ++j) D(i, j) = A(i, j) - A(j, i);
  out[0] = frob(D) / frob(A);
  out[1] = cholesky_ok(A) ? 1.0 : 0.0;
}

/// test_assembly.cpp:40-105: condensation equals the dense Schur complement
/// of the full uncondensed system (gradient variable included).
/// out: [rel gap A, rel gap rhs]
void orc_check_dense_schur(double* out) {
  Mesh mesh = retag_outflow(unit_square(1));
  const int k = 2;
  const Real nu = 2.3, beta = 0.7;
  Space V(mesh, k);
  Constraints con = Constraints::build(V, nullptr);
  AsmOpt opt;
  opt.nu = nu;
  opt.beta = beta;
  opt.load = [](const V2& x) { return V2(std::sin(3 * x.x) + x.y, std::cos(2 * x.y) - x.x * x.x); };
  Condensed sys = assemble_condensed(mesh, V, con, opt);
  const int ns = ref_data(k).ns(), no = V.n_int(), np = ns - 1;
  const Index nco = V.n_compound(), nell = Index(4 * ns) * mesh.ne(), nint = Index(no) * mesh.ne(),
              npp = Index(np) * mesh.ne();
  const Index N = nco + nell + nint + npp;
  Mat K{static_cast<int>(N), static_cast<int>(N)};
  Vec r(N, 0.0);
  AsmOpt mo = opt;
  mo.nu = 0.0;
  for (int e = 0; e < mesh.ne(); ++e) {
    ElemCtx cx(mesh, V, e);
    LocalBlocks b = local_blocks(cx, e, mo);
    std::vector<Index> vd(cx.nv);
    for (int a = 0; a < cx.nc; ++a) vd[a] = cx.gdof[a];
    for (int j = 0; j < no; ++j) vd[cx.nc + j] = nco + nell + Index(e) * no + j;
    const Index ell0 = nco + Index(e) * 4 * ns, p0 = nco + nell + nint + Index(e) * np;
    for (int rr = 0; rr < 4 * ns; ++rr) {
      K(int(ell0 + rr), int(ell0 + rr)) += cx.geo.detJ / nu;
      for (int a = 0; a < cx.nv; ++a) K(int(ell0 + rr), int(vd[a])) += b.C(rr, a);
    }
    for (int a = 0; a < cx.nv; ++a) {
      for (int rr = 0; rr < 4 * ns; ++rr) K(int(vd[a]), int(ell0 + rr)) -= b.C(rr, a);
      for (int c = 0; c < cx.nv; ++c) K(int(vd[a]), int(vd[c])) += b.A(a, c);
      for (int m = 0; m < np; ++m) K(int(vd[a]), int(p0 + m)) -= b.P(m, a);
      r[vd[a]] += b.rhs[a];
    }
    for (int m = 0; m < np; ++m)
      for (int a = 0; a < cx.nv; ++a) K(int(p0 + m), int(vd[a])) -= b.P(m, a);
  }
  const int nl = int(N - nco), nc = int(nco);
  Mat Kll(nl, nl), Klc(nl, nc), Kcl(nc, nl);
  for (int i = 0; i < nl; ++i)
    for (int j = 0; j < nl; ++j) Kll(i, j) = K(nc + i, nc + j);
  for (int i = 0; i < nl; ++i)
    for (int j = 0; j < nc; ++j) Klc(i, j) = K(nc + i, j), Kcl(j, i) = K(j, nc + i);
  FullLU lu(Kll);
  Mat S(nc, nc);
  {
    Mat X(nl, nc);
    for (int j = 0; j < nc; ++j) {
      Vec col(nl);
      for (int i = 0; i < nl; ++i) col[i] = Klc(i, j);
      Vec s = lu.solve(col);
      for (int i = 0; i < nl; ++i) X(i, j) = s[i];
    }
    Mat KX = matmul(Kcl, X);
    for (int i = 0; i < nc; ++i)
      for (int j = 0; j < nc; ++j) S(i, j) = K(i, j) - KX(i, j);
  }
  Vec rl(nl);
  for (int i = 0; i < nl; ++i) rl[i] = r[nc + i];
  Vec y = lu.solve(rl);
  Vec ky = matvec(Kcl, y);
  Vec rs(nc);
  for (int i = 0; i < nc; ++i) rs[i] = r[i] - ky[i];
  Mat A = sys.A.dense();
  Mat D(nc, nc);
  for (int i = 0; i < nc; ++i)
    for (int j = 0; j < nc; ++j) D(i, j) = S(i, j) - A(i, j);
  Vec dr(nc);
  for (int i = 0; i < nc; ++i) dr[i] = rs[i] - sys.rhs[i];
  out[0] = frob(D) / frob(A);
  out[1] = norm(dr) / norm(rs);
}

/// test_assembly.cpp:107-126: constant velocity reproduced via boundary data.
/// out[k]: max error for k = 0..2
void orc_check_constant_velocity(double* out) {
  Mesh mesh = unit_square(2);
  const V2 c(0.8, -0.55);
  for (int k = 0; k <= 2; ++k) {
    Space V(mesh, k);
    Constraints con = Constraints::build(V, [c](const V2&) { return c; });
    AsmOpt opt;
    opt.nu = 1.3;
    opt.beta = 0.9;
    opt.load = [c](const V2&) { return c * 0.9; };
    Condensed sys = assemble_condensed(mesh, V, con, opt);
    Vec u = LU(sys.A.dense()).solve(sys.rhs);
    HDGVel ex = interpolate_hdg(mesh, k, [c](const V2&) { return c; });
    Vec ef = con.to_free(ex.compound);
    Real m = 0;
    for (std::size_t i = 0; i < u.size(); ++i) m = std::max(m, std::abs(u[i] - ef[i]));
    for (Real v : ex.interior) m = std::max(m, std::abs(v));
    out[k] = m;
  }
}

/// test_assembly.cpp:128-162: linear trace-free field recovers interior,
/// zero pressure modes and gradient -nu b. out: max errors [interior, p, grad] over k=1..3
void orc_check_linear_recovery(double* out) {
  Mesh mesh = retag_outflow(unit_square(2));
  const Real nu = 0.8, beta = 1.1;
  const Real b[2][2] = {{0.3, 0.7}, {0.4, -0.3}};
  const V2 a0(0.2, -0.1);
  auto field = [&](const V2& x) { return V2(a0.x + b[0][0] * x.x + b[0][1] * x.y, a0.y + b[1][0] * x.x + b[1][1] * x.y); };
  out[0] = out[1] = out[2] = 0;
  for (int k = 1; k <= 3; ++k) {
    Space V(mesh, k);
    HDGVel u = interpolate_hdg(mesh, k, field);
    AsmOpt opt;
    opt.nu = nu;
    opt.beta = beta;
    opt.load = [&](const V2& x) { return field(x) * beta; };
    LocalSolution loc = recover_locals(mesh, V, opt, u.compound);
    const auto& sc = ref_data(k).scalar;
    const int ns = int(sc.size());
    for (int e = 0; e < mesh.ne(); ++e) {
      for (int j = 0; j < V.n_int(); ++j)
        out[0] = std::max(out[0], std::abs(loc.interior[V.interior(e, j)] - u.interior[V.interior(e, j)]));
      for (int m = 0; m < ns - 1; ++m) out[1] = std::max(out[1], std::abs(loc.p_ortho[std::size_t(e) * (ns - 1) + m]));
      for (int comp = 0; comp < 4; ++comp) {
        Real v = 0;
        for (int m = 0; m < ns; ++m) v += loc.grad(comp * ns + m, e) * sc[m].eval(0.31, 0.29);
        out[2] = std::max(out[2], std::abs(v + nu * b[comp / 2][comp % 2]));
      }
    }
  }
}

/// test_assembly.cpp:164-194: divergence row and grad-div penalty versus
/// quadrature. out: [max |Bx - int div|, max rel penalty gap]
void orc_check_grad_div(double* out) {
  Mesh mesh = retag_outflow(unit_square(2));
  std::mt19937 rng(11);
  std::uniform_real_distribution<Real> dist(-1, 1);
  out[0] = out[1] = 0;
  for (int k = 0; k <= 2; ++k) {
    Space V(mesh, k);
    Constraints con = Constraints::build(V, nullptr);
    Csr B = divergence_rows(V);
    Csr D = grad_div(V, con, Vec(V.n_compound(), 0.0), nullptr);
    Vec x(V.n_compound());
    for (auto& v : x) v = dist(rng);
    Vec interior(V.n_interior());
    for (auto& v : interior) v = dist(rng);
    Vec Bx = B.mul(x);
    const RefData& rd = ref_data(k);
    Real quad = 0;
    for (int e = 0; e < mesh.ne(); ++e) {
      Geo geo(mesh, e);
      Vec coeff(rd.rt.dim, 0.0);
      for (int le = 0; le < 3; ++le)
        for (int i = 0; i <= k; ++i) coeff[rd.rt.facet_fn(le, i)] = x[V.flux(geo.facet[le], i)] * geo.rt_factor(le, i);
      for (int j = 0; j < V.n_int(); ++j) coeff[rd.rt.interior_fn(j)] = interior[V.interior(e, j)];
      Real di = 0;
      for (int q = 0; q < rd.nq(); ++q) {
        Real dq = 0;
        for (int f = 0; f < rd.rt.dim; ++f) dq += rd.vdiv(q, f) * coeff[f];
        di += rd.vol.wts[q] * 2.0 * mesh.area(e) * dq / geo.detJ;
      }
      out[0] = std::max(out[0], std::abs(Bx[e] - di));
      quad += di * di / mesh.area(e);
    }
    // D acts on free DOFs; with no constraints all compound DOFs are free
    // except the Dirichlet-tagged ones (none after retagging).
    Vec xf = con.to_free(x);
    Real pen = dot(xf, D.mul(xf));
    out[1] = std::max(out[1], std::abs(pen - quad) / std::abs(quad));
  }
}

/// test_assembly.cpp:196-219: Picard and Newton share the residual. out: max diff
double orc_check_picard_newton() {
  Mesh mesh = unit_square(2);
  const int k = 1;
  Space V(mesh, k);
  HDGVel st = interpolate_hdg(mesh, k, [](const V2& x) { return V2(0.6 + x.y * (1 - x.y), -0.3 + std::sin(2 * x.x)); });
  AsmOpt base;
  base.nu = 0.05;
  base.beta = 0.2;
  base.load = [](const V2& x) { return V2(1 - x.y, x.x); };
  base.advection = &st;
  AsmOpt nt = base;
  nt.newton = true;
  Real m = 0;
  for (int e = 0; e < mesh.ne(); ++e) {
    ElemCtx cx(mesh, V, e);
    LocalBlocks bp = local_blocks(cx, e, base), bn = local_blocks(cx, e, nt);
    Vec x = cx.local_velocity(st, e);
    Vec rp = matvec(bp.A, x), rn = matvec(bn.A, x);
    for (int i = 0; i < cx.nv; ++i) m = std::max(m, std::abs((rp[i] - bp.rhs[i]) - (rn[i] - bn.rhs[i])));
  }
  return m;
}

/// test_postprocess.cpp:159-225: post-processing preserves element means and
/// satisfies its weak gradient equation, for random normal(0,1) data drawn by
/// std::mt19937(11) in the reference's order (compound, interior, gradient
/// coefficients column by column). out[0] max |mean(u*) - mean(u_h)|,
/// out[1] max per-element residual norm, evaluated at the error rule.
void orc_check_postprocess_weak(double* out) {
  Mesh mesh = unit_square(2);
  const int k = 2;
  Space V(mesh, k);
  const Real nu = 1.3;
  std::mt19937 rng(11);
  std::normal_distribution<Real> coef(0.0, 1.0);
  Vec compound(V.n_compound()), interior(V.n_interior());
  for (auto& v : compound) v = coef(rng);
  for (auto& v : interior) v = coef(rng);
  const RefData& rd = ref_data(k);
  const int ns = rd.ns();
  std::vector<Real> grad(std::size_t(mesh.ne()) * 4 * ns);
  for (auto& v : grad) v = coef(rng);
  std::vector<Real> post = postprocess_velocity(mesh, V, nu, compound, interior, grad);
  const PostTables& pt = post_tables(k);
  const int nh = pt.ns_hi;
  Real mean_err = 0, res_max = 0;
  for (int e = 0; e < mesh.ne(); ++e) {
    ElemCtx cx(mesh, V, e);
    const Vec c = local_rt(cx, V, compound, interior, e);
    const Geo& g = cx.geo;
    Real ms[2] = {0, 0}, mh[2] = {0, 0};
    std::vector<Real> res(2 * nh, 0.0);
    for (std::size_t q = 0; q < pt.err.pts.size(); ++q) {
      const Real w = pt.err.wts[q] * g.detJ;
      const V2 xh = pt.err.pts[q];
      Real hx = 0, hy = 0;
      for (int r = 0; r < cx.nrt; ++r) {
        hx += rd.rt.val[r][0].eval(xh.x, xh.y) * c[r];
        hy += rd.rt.val[r][1].eval(xh.x, xh.y) * c[r];
      }
      const V2 uh = g.applyJ(hx, hy) / g.detJ;
      mh[0] += w * uh.x;
      mh[1] += w * uh.y;
      std::vector<Real> gx(nh), gy(nh), hv(nh);
      for (int s = 0; s < nh; ++s) {
        hv[s] = pt.hi[s].eval(xh.x, xh.y);
        const Real a = pt.hi_grad[s][0].eval(xh.x, xh.y), b = pt.hi_grad[s][1].eval(xh.x, xh.y);
        gx[s] = g.Ji[0][0] * a + g.Ji[1][0] * b;
        gy[s] = g.Ji[0][1] * a + g.Ji[1][1] * b;
      }
      Real L[2][2];
      for (int comp = 0; comp < 4; ++comp) {
        Real v = 0;
        for (int m = 0; m < ns; ++m) v += rd.scalar[m].eval(xh.x, xh.y) * grad[(std::size_t(e) * 4 + comp) * ns + m];
        L[comp / 2][comp % 2] = v;
      }
      for (int i = 0; i < 2; ++i) {
        const Real* pc = &post[std::size_t(e) * 2 * nh + i * nh];
        Real us = 0, gsx = 0, gsy = 0;
        for (int s = 0; s < nh; ++s) {
          us += hv[s] * pc[s];
          gsx += gx[s] * pc[s];
          gsy += gy[s] * pc[s];
        }
        ms[i] += w * us;
        const Real tx = gsx + L[i][0] / nu, ty = gsy + L[i][1] / nu;
        for (int s = 0; s < nh; ++s) res[i * nh + s] += w * (gx[s] * tx + gy[s] * ty);
      }
    }
    mean_err = std::max(mean_err, std::hypot(ms[0] - mh[0], ms[1] - mh[1]));
    Real r2 = 0;
    for (Real v : res) r2 += v * v;
    res_max = std::max(res_max, std::sqrt(r2));
  }
  out[0] = mean_err;
  out[1] = res_max;
}

/// test_assembly.cpp:221-240: upwind transport sees boundary data. out: max err
double orc_check_upwind_lifting() {
  Mesh mesh = unit_square(2);
  Space V(mesh, 0);
  Constraints con = Constraints::build(V, [](const V2&) { return V2(1.0, 0.0); });
  HDGVel w = interpolate_hdg(mesh, 0, [](const V2&) { return V2(1.0, 0.0); });
  AsmOpt opt;
  opt.nu = 0.1;
  opt.advection = &w;
  Condensed sys = assemble_condensed(mesh, V, con, opt);
  Vec u = LU(sys.A.dense()).solve(sys.rhs);
  Vec ref = con.to_free(w.compound);
  Real m = 0;
  for (std::size_t i = 0; i < u.size(); ++i) m = std::max(m, std::abs(u[i] - ref[i]));
  return m;
}

/// test_equivalence.cpp:34-81 and acceptance.cpp:69-110: condensed k=0
/// operator (+ penalty) and load are congruent to the CR midpoint scheme.
/// mesh_kind 0: unit_square(base) refined `refine` times; 1: step_mesh(base).
/// bc_kind: 1 lid on y=1 (acceptance), 2 lid everywhere (test_equivalence).
/// load_kind: 4 smooth test load, 6 manufactured Stokes load (not used).
/// out: [gap A, gap rhs, solution gap]
void orc_check_cr_equivalence(int mesh_kind, int base, int refine_times, double nu, double beta, double inv_eps,
                              int bc_kind, double* out) {
  Mesh mesh = mesh_kind == 0 ? unit_square(base) : step_domain(base);
  for (int r = 0; r < refine_times; ++r) {
    RefineMaps m;
    mesh = refine(mesh, m);
  }
  Field g = bc_kind == 1 ? Field([](const V2& x) { return x.y > 1.0 - 1e-12 ? V2(4 * x.x * (1 - x.x), 0.0) : V2(0, 0); })
                         : Field([](const V2& x) { return V2(4 * x.x * (1 - x.x), 0.0); });
  Field load = [](const V2& x) { return V2(std::sin(3 * x.x) - x.y, std::cos(2 * x.y) + x.x * x.y); };
  Space V(mesh, 0);
  Constraints con = Constraints::build(V, g);
  AsmOpt opt;
  opt.nu = nu;
  opt.beta = beta;
  opt.load = load;
  Condensed sys = assemble_condensed(mesh, V, con, opt);
  Vec rd;
  Csr D = grad_div(V, con, con.g_full, &rd);
  Mat Ah = sys.A.add(D, inv_eps).dense();
  Vec rh = sys.rhs;
  for (std::size_t i = 0; i < rh.size(); ++i) rh[i] += inv_eps * rd[i];
  cr::System crs = cr::assemble(mesh, nu, beta, inv_eps, load, g);
  Mat F = cr::from_compound(V).dense();
  const int nr = int(crs.free_to_full.size()), nc = int(con.free_to_full.size());
  Mat P(nr, nc);
  for (int i = 0; i < nr; ++i)
    for (int j = 0; j < nc; ++j) P(i, j) = F(int(crs.free_to_full[i]), int(con.free_to_full[j]));
  Mat Am = matmul(matmul(P.t(), crs.A.dense()), P);
  Vec rm = matvec(P.t(), crs.rhs);
  Mat DA(nc, nc);
  for (int i = 0; i < nc; ++i)
    for (int j = 0; j < nc; ++j) DA(i, j) = Ah(i, j) - Am(i, j);
  Vec dr(nc);
  for (int i = 0; i < nc; ++i) dr[i] = rh[i] - rm[i];
  out[0] = frob(DA) / frob(Ah);
  out[1] = norm(dr) / norm(rh);
  Vec uh = LU(Ah).solve(rh);
  Vec uc = LU(crs.A.dense()).solve(crs.rhs);
  Vec pu = matvec(P, uh);
  for (int i = 0; i < nr; ++i) pu[i] -= uc[i];
  out[2] = norm(pu) / norm(uc);
}

/// test_transfer.cpp:38-49 (linear reproduction, unit square + step),
/// :90-113 (interior patches), :115-158 (corrected P), :160-182 (embedding),
/// :184-198 (advection restriction).
/// out: [lin gap square, lin gap step, interior patches ok, max interior
/// residual row / ref, max non-interior row change, d_avg/|u|^2, d_corr/d_avg,
/// |E^T E - I|, |E u0 - u3|/|u3|, |E^T v3 - v0|/|v0|, restrict gap, lowest-order gap]
void orc_check_transfers(double* out) {
  auto lin = [](const V2& x) { return V2(0.3 - 0.7 * x.x + 1.2 * x.y, -0.4 + 0.9 * x.x + 0.5 * x.y); };
  Field zero = [](const V2&) { return V2(0, 0); };
  for (int which = 0; which < 2; ++which) {
    Mesh cm = retag_outflow(which == 0 ? unit_square(2) : step_domain(2));
    RefineMaps maps;
    Mesh fm = refine(cm, maps);
    Space Vc(cm, 0), Vf(fm, 0);
    Constraints cc = Constraints::build(Vc, zero), cf = Constraints::build(Vf, zero);
    Csr P = averaging_transfer(Vc, cc, Vf, cf, maps);
    Vec uc = cc.to_free(interpolate_hdg(cm, 0, lin).compound);
    Vec uf = cf.to_free(interpolate_hdg(fm, 0, lin).compound);
    Vec pu = P.mul(uc);
    for (std::size_t i = 0; i < pu.size(); ++i) pu[i] -= uf[i];
    out[which] = norm(pu) / norm(uf);
  }
  Mesh cm = unit_square(2);
  RefineMaps maps;
  Mesh fm = refine(cm, maps);
  Space Vc(cm, 0), Vf(fm, 0);
  Constraints cc = Constraints::build(Vc, zero), cf = Constraints::build(Vf, zero);
  auto blocks = interior_patch_dofs(Vf, cf, maps);
  {
    bool ok = int(blocks.size()) == cm.ne();
    std::vector<int> seen(cf.n_free, 0);
    for (const auto& b : blocks) {
      ok = ok && b.size() == 6;
      for (Index d : b) {
        ok = ok && d >= 0 && d < cf.n_free;
        if (d >= 0 && d < cf.n_free) ++seen[d];
      }
    }
    int medial = 0, covered = 0;
    for (int c : maps.fine_class) medial += c == kInteriorOfCoarse;
    for (int s : seen) { ok = ok && s <= 1; covered += s; }
    ok = ok && medial == 3 * cm.ne() && covered == 6 * cm.ne();
    out[2] = ok ? 1.0 : 0.0;
  }
  const Real inv_eps = 1e6;
  AsmOpt opt;
  Condensed sys = assemble_condensed(fm, Vf, cf, opt);
  Csr Df = grad_div(Vf, cf, cf.g_full, nullptr);
  Csr A = sys.A.add(Df, inv_eps);
  Csr Iavg = averaging_transfer(Vc, cc, Vf, cf, maps);
  Csr P = corrected_prolongation(Iavg, A, blocks);
  std::vector<char> is_t(cf.n_free, 0);
  for (const auto& b : blocks)
    for (Index d : b) is_t[d] = 1;
  Mat Ravg = spmul(A, Iavg).dense(), R = spmul(A, P).dense();
  Real ref = 0;
  for (Real v : Ravg.a) ref = std::max(ref, std::abs(v));
  Mat Pd = P.dense(), Id = Iavg.dense();
  Real worst_t = 0, worst_nt = 0;
  for (int r = 0; r < R.r; ++r)
    for (int c = 0; c < R.c; ++c) {
      if (is_t[r]) worst_t = std::max(worst_t, std::abs(R(r, c)) / ref);
      else worst_nt = std::max(worst_nt, std::abs(Pd(r, c) - Id(r, c)));
    }
  out[3] = worst_t;
  out[4] = worst_nt;
  {
    // divergence-free coarse correction: kernel of the free coarse divergence rows
    Mat Bc = divergence_rows(Vc).dense();
    Mat Bf(cm.ne(), int(cc.n_free));
    for (Index j = 0; j < cc.n_free; ++j)
      for (int i = 0; i < cm.ne(); ++i) Bf(i, int(j)) = Bc(i, int(cc.free_to_full[j]));
    SVD sv(Bf);
    int n = Bf.c, rank = 0;
    for (Real s : sv.s) rank += s > 1e-12 * sv.s[0];
    Vec c(n, 0.0);
    for (int j = rank; j < n; ++j)
      for (int i = 0; i < n; ++i) c[i] += sv.V(i, j);
    Vec ua = Iavg.mul(c), ucr = P.mul(c);
    Real da = dot(ua, Df.mul(ua)), dc = dot(ucr, Df.mul(ucr));
    out[5] = da / dot(ua, ua);
    out[6] = dc / da;
  }
  {
    Space V0(cm, 0), V3(cm, 3);
    Constraints c0 = Constraints::build(V0, zero), c3 = Constraints::build(V3, zero);
    Csr E = order_embedding(V0, c0, V3, c3);
    Mat ETE = matmul(E.transpose().dense(), E.dense());
    Real g = 0;
    for (int i = 0; i < ETE.r; ++i)
      for (int j = 0; j < ETE.c; ++j) g = std::max(g, std::abs(ETE(i, j) - (i == j ? 1.0 : 0.0)));
    out[7] = g;
    auto cst = [](const V2&) { return V2(0.4, -0.8); };
    Vec u0 = c0.to_free(interpolate_hdg(cm, 0, cst).compound), u3 = c3.to_free(interpolate_hdg(cm, 3, cst).compound);
    Vec eu = E.mul(u0);
    for (std::size_t i = 0; i < eu.size(); ++i) eu[i] -= u3[i];
    out[8] = norm(eu) / norm(u3);
    auto fl = [](const V2& x) { return V2(0.4 + 0.6 * x.x, -0.8 + 0.6 * x.y); };
    Vec v0 = c0.to_free(interpolate_hdg(cm, 0, fl).compound), v3 = c3.to_free(interpolate_hdg(cm, 3, fl).compound);
    Vec ev = E.transpose().mul(v3);
    for (std::size_t i = 0; i < ev.size(); ++i) ev[i] -= v0[i];
    out[9] = norm(ev) / norm(v0);
  }
  {
    auto field = [](const V2& x) { return V2(0.2 + x.x * x.y - x.y * x.y, -0.5 * x.x * x.x + 0.3 * x.y); };
    HDGVel wf = interpolate_hdg(fm, 0, field);
    HDGVel wc = restrict_advection(wf, Vc, maps);
    HDGVel ref2 = interpolate_hdg(cm, 0, field);
    Vec d(wc.compound.size());
    for (std::size_t i = 0; i < d.size(); ++i) d[i] = wc.compound[i] - ref2.compound[i];
    out[10] = norm(d) / norm(ref2.compound);
    HDGVel w2 = interpolate_hdg(cm, 2, field);
    HDGVel w0 = lowest_order_advection(w2, Vc);
    for (std::size_t i = 0; i < d.size(); ++i) d[i] = w0.compound[i] - ref2.compound[i];
    out[11] = norm(d) / norm(ref2.compound);
  }
}

}  // extern "C"
