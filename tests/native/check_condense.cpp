// TEST INFRASTRUCTURE: host build of the product's element-condensation
// routine (paper_2303_06762_b200/csrc/kernels/condense.cuh, compiled with
// SYNC() as a no-op and one "thread") checked element by element against the
// CPU oracle, for Stokes (mass + load), Oseen (upwinded convection about a
// wind interpolated independently by each side), the Newton linearisation
// about that wind, and the pseudo-time mass-field load. Also checks that the
// product mesh numbering equals the oracle's.
#define SYNC()
#include <cstdio>
#include <memory>

#include "../../oracle/orc_mg.hpp"
#include "../../paper_2303_06762_b200/csrc/host/basis.hpp"
#include "../../paper_2303_06762_b200/csrc/host/plan.hpp"
#include "../../paper_2303_06762_b200/csrc/host/wind.hpp"

using namespace hpmg;

int main() {
  double worst_rel = 0, worst_rhs = 0, worst_adv = 0, worst_newton = 0, worst_newton_rhs = 0, worst_mass = 0;
  double worst_recover = 0;
  int bad_mesh = 0;
  // the config-5 wind (tangential to the boundary, vanishing at the corners:
  // the upwind switch sees round-off-level w.n) and a shifted variant
  double shift = 0.0;
  auto wind = [&](double x, double y, double* out) {
    const double s = std::sin(M_PI * x), t = std::sin(M_PI * y);
    out[0] = M_PI * s * s * std::sin(2 * M_PI * y) + 0.3 * shift;
    out[1] = -M_PI * std::sin(2 * M_PI * x) * t * t - 0.2 * shift;
  };
  for (int kk = 0; kk < 8; ++kk) {
    const int k = kk % 4;
    shift = kk < 4 ? 0.0 : 1.0;
    auto T = host::build_ref_tensors(k);
    RefT R{T->k,        T->nfd,     T->nrt,      T->no,       T->ns,       T->nc,       T->nv,
           T->G.data(), T->Mm.data(), T->Dv.data(), T->Lv.data(), T->Ev.data(), T->Tv.data(), T->vval.data(),
           T->qw.data(), T->nq,     T->vjac.data(), T->evp.data(), T->ew.data(), T->eleg.data(), T->nqe};
    orc::Mesh om = orc::unit_square(2);
    host::TriMesh hm = host::unit_square(2);
    for (int lev = 0; lev < 2; ++lev) {
      orc::RefineMaps rm;
      om = orc::refine(om, rm);
      host::Refinement hr;
      hm = host::refine(hm, hr);
    }
    // mesh numbering identical
    if (om.nf() != hm.nf() || om.ne() != hm.ne()) bad_mesh++;
    for (int f = 0; f < om.nf(); ++f)
      if (om.fc[f].a != hm.fa[f] || om.fc[f].b != hm.fb[f] || om.fc[f].tag != hm.ftag[f]) bad_mesh++;
    for (int e = 0; e < om.ne(); ++e)
      for (int i = 0; i < 3; ++i)
        if (om.el[e].facet[i] != hm.ef[e][i] || om.el[e].sigma[i] != hm.esig[e][i] || om.el[e].rho[i] != hm.erho[e][i])
          bad_mesh++;
    orc::Space V(om, k);
    orc::HDGVel ow = orc::interpolate_hdg(om, k, [&](const orc::V2& x) {
      double o[2];
      wind(x.x, x.y, o);
      return orc::V2(o[0], o[1]);
    });
    host::HdgField hw = host::interpolate_hdg(hm, k, *T, wind);
    std::vector<double> xw_all = host::local_wind(hm, k, hw);
    // modes: 0 Stokes + mass + load, 1 Stokes, 2 Oseen, 3 Newton, 4 pseudo-time mass field + load
    for (int mode = 0; mode < 5; ++mode) {
      orc::AsmOpt opt;
      opt.nu = mode >= 2 ? 0.05 : 1.3;
      opt.beta = mode == 0 ? 0.7 : 0.0;
      const double F[2] = {0.37, -0.81};
      if (mode == 0 || mode == 4) opt.load = [&](const orc::V2&) { return orc::V2(F[0], F[1]); };
      if (mode == 2 || mode == 3) opt.advection = &ow;
      if (mode == 3) opt.newton = true;
      if (mode == 4) {
        opt.mass_coef = 2.5;
        opt.mass_field = &ow;
      }
      CondenseParams prm{opt.nu, opt.beta + opt.mass_coef, (mode == 0 || mode == 4) ? 1 : 0, mode == 3 ? 1 : 0,
                         opt.mass_coef};
      int nz = T->no + T->ns - 1;
      std::vector<double> scratch(condense_scratch(T->ns, T->nv, T->nc, nz, T->nrt, T->nq, T->nqe));
      std::vector<double> Ac(T->nc * T->nc), rc(T->nc);
      // load vectors are compared against the mode's global scale: elements
      // where the wind vanishes carry round-off-only Newton loads
      double mode_rmx = 0, mode_rdf = 0;
      for (int e = 0; e < om.ne(); ++e) {
        orc::ElemCtx cx(om, V, e);
        orc::LocalBlocks b = orc::local_blocks(cx, e, opt);
        orc::Mat oAc;
        orc::Vec orc_;
        orc::condense(cx, b, oAc, orc_);
        ElemGeo g = host::element_geometry(hm, e);
        condense_element(0, 1, R, g, prm, F, scratch.data(), Ac.data(), rc.data(), nullptr, nullptr, nullptr,
                         (mode == 2 || mode == 3) ? &xw_all[size_t(e) * T->nv] : nullptr,
                         mode == 4 ? &xw_all[size_t(e) * T->nv] : nullptr);
        double mx = 0, df = 0, rmx = 0, rdf = 0;
        for (int i = 0; i < T->nc; ++i) {
          for (int j = 0; j < T->nc; ++j) {
            mx = std::max(mx, std::abs(oAc(i, j)));
            df = std::max(df, std::abs(oAc(i, j) - Ac[i * T->nc + j]));
          }
          rmx = std::max(rmx, std::abs(orc_[i]));
          rdf = std::max(rdf, std::abs(orc_[i] - rc[i]));
        }
        if (mode == 2) worst_adv = std::max(worst_adv, df / mx);
        else if (mode == 3) worst_newton = std::max(worst_newton, df / mx);
        else worst_rel = std::max(worst_rel, df / mx);
        mode_rmx = std::max(mode_rmx, rmx);
        mode_rdf = std::max(mode_rdf, rdf);
      }
      if (mode_rmx > 0) {
        const double r = mode_rdf / mode_rmx;
        if (mode == 3) worst_newton_rhs = std::max(worst_newton_rhs, r);
        else if (mode == 4) worst_mass = std::max(worst_mass, r);
        else worst_rhs = std::max(worst_rhs, r);
      }
    }
    // recovery mode (recover_locals, assembly.hpp:513-549) under the Oseen and
    // Newton linearisations: gradient variable and pressure modes are
    // basis-independent
    for (int mode = 2; mode < 4; ++mode) {
      orc::AsmOpt opt;
      opt.nu = 0.05;
      opt.advection = &ow;
      opt.newton = mode == 3;
      CondenseParams prm{opt.nu, 0.0, 0, mode == 3 ? 1 : 0, 0.0};
      orc::Vec comp(V.n_compound());
      for (std::size_t i = 0; i < comp.size(); ++i) comp[i] = std::sin(0.7 * double(i) + 0.3);
      orc::LocalSolution ls = orc::recover_locals(om, V, opt, comp);
      const int nz = T->no + T->ns - 1;
      std::vector<double> scratch(condense_scratch(T->ns, T->nv, T->nc, nz, T->nrt, T->nq, T->nqe));
      std::vector<double> xc(T->nc), z(nz + 1), gr(4 * T->ns);
      double gmx = 0, gdf = 0, pmx = 0, pdf = 0;
      for (int e = 0; e < om.ne(); ++e) {
        orc::ElemCtx cx(om, V, e);
        for (int a = 0; a < T->nc; ++a) xc[a] = comp[cx.gdof[a]];
        ElemGeo g = host::element_geometry(hm, e);
        condense_element(0, 1, R, g, prm, nullptr, scratch.data(), nullptr, nullptr, xc.data(), z.data(), gr.data(),
                         &xw_all[size_t(e) * T->nv]);
        for (int r = 0; r < 4 * T->ns; ++r) {
          gmx = std::max(gmx, std::abs(ls.grad(r, e)));
          gdf = std::max(gdf, std::abs(ls.grad(r, e) - gr[r]));
        }
        for (int m = 0; m < T->ns - 1; ++m) {
          const double po = ls.p_ortho[std::size_t(e) * (T->ns - 1) + m];
          pmx = std::max(pmx, std::abs(po));
          pdf = std::max(pdf, std::abs(po - z[T->no + m]));
        }
      }
      const double gr_rel = gmx > 0 ? gdf / gmx : 0, p_rel = pmx > 0 ? pdf / pmx : 0;
      worst_recover = std::max(worst_recover, std::max(gr_rel, p_rel));
      printf("k=%d shift %.0f recovery mode %d: grad rel %.3e pressure rel %.3e\n", k, shift, mode, gr_rel, p_rel);
    }
    printf("k=%d shift %.0f worst Ac rel %.3e rhs rel %.3e advected Ac rel %.3e newton Ac rel %.3e rhs rel %.3e mass-field rhs rel %.3e\n",
           k, shift, worst_rel, worst_rhs, worst_adv, worst_newton, worst_newton_rhs, worst_mass);
  }
  printf("mesh mismatches %d\n", bad_mesh);
  const bool ok = worst_rel < 1e-12 && worst_rhs < 1e-12 && worst_adv < 1e-11 && worst_newton < 1e-11 &&
                  worst_newton_rhs < 1e-11 && worst_mass < 1e-12 && worst_recover < 1e-11 && bad_mesh == 0;
  printf("RESULT %s\n", ok ? "PASS" : "FAIL");
  return ok ? 0 : 1;
}
