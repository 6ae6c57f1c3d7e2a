// TEST INFRASTRUCTURE: host build of the product's element-condensation
// routine (paper_2303_06762_b200/csrc/kernels/condense.cuh, compiled with
// SYNC() as a no-op and one "thread") checked element by element against the
// CPU oracle. Also checks that the product mesh numbering equals the oracle's.
#define SYNC()
#include <cstdio>
#include <memory>

#include "../../oracle/orc_mg.hpp"
#include "../../paper_2303_06762_b200/csrc/host/basis.hpp"
#include "../../paper_2303_06762_b200/csrc/host/plan.hpp"

using namespace hpmg;

int main() {
  double worst_rel = 0, worst_rhs = 0;
  int bad_mesh = 0;
  for (int k = 0; k <= 3; ++k) {
    auto T = host::build_ref_tensors(k);
    RefT R{T->k, T->nfd, T->nrt, T->no, T->ns, T->nc, T->nv, T->G.data(), T->Mm.data(), T->Dv.data(),
           T->Lv.data(), T->Ev.data(), T->Tv.data(), T->vval.data(), T->qw.data(), T->nq};
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
    for (int mode = 0; mode < 2; ++mode) {
      orc::AsmOpt opt;
      opt.nu = 1.3;
      opt.beta = mode == 0 ? 0.7 : 0.0;
      const double F[2] = {0.37, -0.81};
      if (mode == 0) opt.load = [&](const orc::V2&) { return orc::V2(F[0], F[1]); };
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
        condense_element(0, 1, R, g, prm, F, scratch.data(), Ac.data(), rc.data());
        double mx = 0, df = 0, rmx = 0, rdf = 0;
        for (int i = 0; i < T->nc; ++i) {
          for (int j = 0; j < T->nc; ++j) {
            mx = std::max(mx, std::abs(oAc(i, j)));
            df = std::max(df, std::abs(oAc(i, j) - Ac[i * T->nc + j]));
          }
          rmx = std::max(rmx, std::abs(orc_[i]));
          rdf = std::max(rdf, std::abs(orc_[i] - rc[i]));
        }
        worst_rel = std::max(worst_rel, df / mx);
        if (rmx > 0) worst_rhs = std::max(worst_rhs, rdf / rmx);
      }
    }
    printf("k=%d worst Ac rel %.3e rhs rel %.3e\n", k, worst_rel, worst_rhs);
  }
  printf("mesh mismatches %d\n", bad_mesh);
  printf("RESULT %s\n", (worst_rel < 1e-12 && worst_rhs < 1e-12 && bad_mesh == 0) ? "PASS" : "FAIL");
  return (worst_rel < 1e-12 && worst_rhs < 1e-12 && bad_mesh == 0) ? 0 : 1;
}
