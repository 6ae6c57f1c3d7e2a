// TEST INFRASTRUCTURE: host build of the product's element-condensation
// routine (paper_2303_06762_b200/csrc/kernels/condense.cuh, compiled with
// SYNC() as a no-op and one "thread") checked element by element against the
// CPU oracle, for Stokes (mass + load) and Oseen (upwinded convection about a
// wind interpolated independently by each side). Also checks that the
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
  double worst_rel = 0, worst_rhs = 0, worst_adv = 0;
  int bad_mesh = 0;
  auto wind = [](double x, double y, double* out) {
    const double s = std::sin(M_PI * x), t = std::sin(M_PI * y);
    out[0] = M_PI * s * s * std::sin(2 * M_PI * y) + 0.3;
    out[1] = -M_PI * std::sin(2 * M_PI * x) * t * t - 0.2;
  };
  for (int k = 0; k <= 3; ++k) {
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
    for (int mode = 0; mode < 3; ++mode) {
      orc::AsmOpt opt;
      opt.nu = mode == 2 ? 0.05 : 1.3;
      opt.beta = mode == 0 ? 0.7 : 0.0;
      const double F[2] = {0.37, -0.81};
      if (mode == 0) opt.load = [&](const orc::V2&) { return orc::V2(F[0], F[1]); };
      if (mode == 2) opt.advection = &ow;
      CondenseParams prm{opt.nu, opt.beta, mode == 0 ? 1 : 0};
      int nz = T->no + T->ns - 1;
      std::vector<double> scratch(condense_scratch(T->ns, T->nv, T->nc, nz, T->nrt));
      std::vector<double> Ac(T->nc * T->nc), rc(T->nc);
      for (int e = 0; e < om.ne(); ++e) {
        orc::ElemCtx cx(om, V, e);
        orc::LocalBlocks b = orc::local_blocks(cx, e, opt);
        orc::Mat oAc;
        orc::Vec orc_;
        orc::condense(cx, b, oAc, orc_);
        ElemGeo g = host::element_geometry(hm, e);
        condense_element(0, 1, R, g, prm, F, scratch.data(), Ac.data(), rc.data(), nullptr, nullptr, nullptr,
                         mode == 2 ? &xw_all[size_t(e) * T->nv] : nullptr);
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
        else worst_rel = std::max(worst_rel, df / mx);
        if (rmx > 0) worst_rhs = std::max(worst_rhs, rdf / rmx);
      }
    }
    printf("k=%d worst Ac rel %.3e rhs rel %.3e advected Ac rel %.3e\n", k, worst_rel, worst_rhs, worst_adv);
  }
  printf("mesh mismatches %d\n", bad_mesh);
  const bool ok = worst_rel < 1e-12 && worst_rhs < 1e-12 && worst_adv < 1e-11 && bad_mesh == 0;
  printf("RESULT %s\n", ok ? "PASS" : "FAIL");
  return ok ? 0 : 1;
}
