// TEST INFRASTRUCTURE ONLY (see orc_core.hpp). Crouzeix-Raviart known-answer
// scheme, intergrid transfers, vertex-patch smoother, hp-multigrid
// preconditioner, PCG / GMRES and the augmented-Lagrangian Uzawa loop
// (reference inc/cr.hpp, transfer.hpp, smoother.hpp, multigrid.hpp,
// krylov.hpp, uzawa.hpp).
#pragma once

#include <memory>
#include <unordered_map>

#include "orc_assembly.hpp"

namespace orc {

// ------------------------------------------------------------------- CR ----
namespace cr {
inline Index dof(int f, int c) { return 2 * Index(f) + c; }
/// 1 - 2 lambda_opposite (inc/cr.hpp:69-77)
inline Real basis_value(const Mesh& m, int e, int lf, const V2& x) {
  const auto& E = m.el[e];
  V2 p = m.vtx[E.v[lf]], a = m.vtx[E.v[(lf + 1) % 3]], b = m.vtx[E.v[(lf + 2) % 3]];
  Real full = (b - a).x * (p - a).y - (b - a).y * (p - a).x;
  Real part = (b - a).x * (x - a).y - (b - a).y * (x - a).x;
  return 1.0 - 2.0 * part / full;
}
inline V2 basis_gradient(const Mesh& m, int e, int lf) {
  int f = m.el[e].facet[lf];
  return m.fnormal(f) * (Real(m.el[e].sigma[lf]) * m.flen(f) / m.area(e));
}
inline V2 rt0_value(const Mesh& m, int e, int lf, const V2& x) {
  const auto& E = m.el[e];
  return (x - m.vtx[E.v[lf]]) * (Real(E.sigma[lf]) * m.flen(E.facet[lf]) / (2.0 * m.area(e)));
}
struct System {
  Csr A;
  Vec rhs, g_full;
  std::vector<Index> full_to_free, free_to_full;
};
/// Independent midpoint assembly (inc/cr.hpp:108-180).
inline System assemble(const Mesh& m, Real nu, Real beta, Real inv_eps, const Field& load, const Field& g) {
  System s;
  const Index nfull = 2 * Index(m.nf());
  s.g_full.assign(nfull, 0.0);
  s.full_to_free.assign(nfull, -1);
  LineRule glr = line_rule(6);
  for (int f = 0; f < m.nf(); ++f) {
    if (m.fc[f].tag != kDirichlet) {
      for (int c = 0; c < 2; ++c) {
        s.full_to_free[dof(f, c)] = Index(s.free_to_full.size());
        s.free_to_full.push_back(dof(f, c));
      }
      continue;
    }
    if (!g) continue;
    V2 mean;
    for (std::size_t q = 0; q < glr.pts.size(); ++q) mean += g(m.fpoint(f, glr.pts[q])) * (0.5 * glr.wts[q]);
    s.g_full[dof(f, 0)] = mean.x;
    s.g_full[dof(f, 1)] = mean.y;
  }
  const Index nfree = Index(s.free_to_full.size());
  s.rhs.assign(nfree, 0.0);
  TriRule tr = tri_rule(4);
  std::vector<Trip> t;
  for (int e = 0; e < m.ne(); ++e) {
    const auto& E = m.el[e];
    const Real area = m.area(e);
    V2 grad[3], nf[3];
    Real dr[3];
    for (int i = 0; i < 3; ++i) {
      grad[i] = basis_gradient(m, e, i);
      nf[i] = m.fnormal(E.facet[i]);
      dr[i] = Real(E.sigma[i]) * m.flen(E.facet[i]) / area;
    }
    Mat K(6, 6);
    Vec re(6, 0.0);
    auto comp = [](const V2& v, int c) { return c == 0 ? v.x : v.y; };
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        Real visc = nu * area * grad[i].dot(grad[j]);
        for (int c = 0; c < 2; ++c) K(2 * i + c, 2 * j + c) += visc;
        for (int ci = 0; ci < 2; ++ci)
          for (int cj = 0; cj < 2; ++cj)
            K(2 * i + ci, 2 * j + cj) += inv_eps * area * dr[i] * comp(nf[i], ci) * dr[j] * comp(nf[j], cj);
      }
    if (beta != 0.0 || load) {
      for (std::size_t q = 0; q < tr.pts.size(); ++q) {
        V2 xr = tr.pts[q];
        V2 x = m.vtx[E.v[0]] + (m.vtx[E.v[1]] - m.vtx[E.v[0]]) * xr.x + (m.vtx[E.v[2]] - m.vtx[E.v[0]]) * xr.y;
        Real w = tr.wts[q] * 2.0 * area;
        V2 rt[3];
        for (int i = 0; i < 3; ++i) rt[i] = rt0_value(m, e, i, x);
        if (beta != 0.0)
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
              for (int ci = 0; ci < 2; ++ci)
                for (int cj = 0; cj < 2; ++cj)
                  K(2 * i + ci, 2 * j + cj) += beta * w * comp(nf[i], ci) * comp(nf[j], cj) * rt[i].dot(rt[j]);
        if (load) {
          V2 fv = load(x);
          for (int i = 0; i < 3; ++i)
            for (int c = 0; c < 2; ++c) re[2 * i + c] += w * comp(nf[i], c) * fv.dot(rt[i]);
        }
      }
    }
    for (int i = 0; i < 3; ++i)
      for (int ci = 0; ci < 2; ++ci) {
        Index fi = s.full_to_free[dof(E.facet[i], ci)];
        if (fi < 0) continue;
        s.rhs[fi] += re[2 * i + ci];
        for (int j = 0; j < 3; ++j)
          for (int cj = 0; cj < 2; ++cj) {
            Index gj = dof(E.facet[j], cj), fj = s.full_to_free[gj];
            if (fj >= 0) t.push_back({fi, fj, K(2 * i + ci, 2 * j + cj)});
            else s.rhs[fi] -= K(2 * i + ci, 2 * j + cj) * s.g_full[gj];
          }
      }
  }
  s.A = Csr::from_trips(nfree, nfree, t);
  return s;
}
/// Per-facet frame change compound -> midpoint vectors (inc/cr.hpp:184-199).
inline Csr from_compound(const Space& V) {
  const Mesh& m = *V.mesh;
  std::vector<Trip> t;
  for (int f = 0; f < m.nf(); ++f) {
    V2 n = m.fnormal(f), tt = m.ftan(f);
    t.push_back({dof(f, 0), V.flux(f, 0), n.x});
    t.push_back({dof(f, 0), V.tang(f, 0), tt.x});
    t.push_back({dof(f, 1), V.flux(f, 0), n.y});
    t.push_back({dof(f, 1), V.tang(f, 0), tt.y});
  }
  return Csr::from_trips(2 * Index(m.nf()), V.n_compound(), t);
}
}  // namespace cr

// ------------------------------------------------------------- transfer ----
/// CR averaging between free lowest-order spaces (inc/transfer.hpp:19-71).
inline Csr averaging_transfer(const Space& Vc, const Constraints& cc, const Space& Vf, const Constraints& cf,
                              const RefineMaps& maps) {
  const Mesh& cm = *Vc.mesh;
  const Mesh& fm = *Vf.mesh;
  std::vector<Trip> t;
  for (int ff = 0; ff < fm.nf(); ++ff) {
    Index rn = cf.full_to_free[Vf.flux(ff, 0)], rt = cf.full_to_free[Vf.tang(ff, 0)];
    if (rn < 0) continue;
    std::pair<int, Real> sides[2] = {{-1, 0.0}, {-1, 0.0}};
    switch (maps.fine_class[ff]) {
      case kInteriorOfCoarse: sides[0] = {maps.fine_parent_element[ff], 1.0}; break;
      case kOnBoundary: sides[0] = {cm.fc[maps.fine_parent_facet[ff]].elem[0], 1.0}; break;
      default: {
        const auto& pf = cm.fc[maps.fine_parent_facet[ff]];
        sides[0] = {pf.elem[0], 0.5};
        sides[1] = {pf.elem[1], 0.5};
      }
    }
    V2 xm = fm.fmid(ff), nf = fm.fnormal(ff), tf = fm.ftan(ff);
    for (auto [e, w] : sides) {
      if (e < 0) continue;
      for (int i = 0; i < 3; ++i) {
        int fc = cm.el[e].facet[i];
        Real phi = w * cr::basis_value(cm, e, i, xm);
        V2 nc = cm.fnormal(fc), tc = cm.ftan(fc);
        Index cn = cc.full_to_free[Vc.flux(fc, 0)], ct = cc.full_to_free[Vc.tang(fc, 0)];
        if (cn >= 0) {
          t.push_back({rn, cn, phi * nf.dot(nc)});
          t.push_back({rt, ct, phi * tf.dot(tc)});
          t.push_back({rn, ct, phi * nf.dot(tc)});
          t.push_back({rt, cn, phi * tf.dot(nc)});
        }
      }
    }
  }
  return Csr::from_trips(cf.n_free, cc.n_free, t, true);
}

/// (inc/transfer.hpp:75-88)
inline std::vector<std::vector<Index>> interior_patch_dofs(const Space& Vf, const Constraints& cf, const RefineMaps& maps) {
  const Mesh& fm = *Vf.mesh;
  std::vector<std::vector<Index>> blk(maps.elem_children.size());
  for (int ff = 0; ff < fm.nf(); ++ff) {
    if (maps.fine_class[ff] != kInteriorOfCoarse) continue;
    auto& b = blk[maps.fine_parent_element[ff]];
    for (int i = 0; i <= Vf.k; ++i) {
      b.push_back(cf.full_to_free[Vf.flux(ff, i)]);
      b.push_back(cf.full_to_free[Vf.tang(ff, i)]);
    }
  }
  return blk;
}

/// P = I_avg with interior rows replaced by -A_TT^{-1} (A I_avg)_T
/// (inc/transfer.hpp:95-133).
inline Csr corrected_prolongation(const Csr& Iavg, const Csr& A, const std::vector<std::vector<Index>>& blocks) {
  Csr W = spmul(A, Iavg);
  std::vector<char> is_t(Iavg.rows, 0);
  for (const auto& T : blocks)
    for (Index r : T) is_t[r] = 1;
  std::vector<Trip> t;
  // Eigen sums the averaging and the correction triplets into one matrix, so
  // the corrected rows hold I_avg + (-X) entrywise (inc/transfer.hpp:110-131).
  for (Index i = 0; i < Iavg.rows; ++i)
    for (Index p = Iavg.ptr[i]; p < Iavg.ptr[i + 1]; ++p) t.push_back({i, Iavg.idx[p], Iavg.val[p]});
  for (const auto& T : blocks) {
    const int nt = int(T.size());
    if (nt == 0) continue;
    std::vector<Index> cols;
    for (Index r : T)
      for (Index p = W.ptr[r]; p < W.ptr[r + 1]; ++p) cols.push_back(W.idx[p]);
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    if (cols.empty()) continue;
    std::unordered_map<Index, int> loc;
    for (std::size_t j = 0; j < cols.size(); ++j) loc[cols[j]] = int(j);
    Mat Att(nt, nt), Wt(nt, int(cols.size()));
    for (int r = 0; r < nt; ++r) {
      for (int s = 0; s < nt; ++s) Att(r, s) = A.coeff(T[r], T[s]);
      for (Index p = W.ptr[T[r]]; p < W.ptr[T[r] + 1]; ++p) Wt(r, loc[W.idx[p]]) = W.val[p];
    }
    Mat X = LU(Att).solve(Wt);
    for (int r = 0; r < nt; ++r)
      for (std::size_t j = 0; j < cols.size(); ++j) t.push_back({T[r], cols[j], -X(r, int(j))});
  }
  return Csr::from_trips(Iavg.rows, Iavg.cols, t, true);
}

/// Free lowest-order -> free order-k injection of constant facet modes
/// (inc/transfer.hpp:140-158).
inline Csr order_embedding(const Space& V0, const Constraints& c0, const Space& Vk, const Constraints& ck) {
  const Mesh& m = *V0.mesh;
  std::vector<Trip> t;
  for (int f = 0; f < m.nf(); ++f) {
    Index cn = c0.full_to_free[V0.flux(f, 0)], rn = ck.full_to_free[Vk.flux(f, 0)];
    if (cn < 0) continue;
    t.push_back({rn, cn, 1.0});
    t.push_back({ck.full_to_free[Vk.tang(f, 0)], c0.full_to_free[V0.tang(f, 0)], 1.0});
  }
  return Csr::from_trips(ck.n_free, c0.n_free, t);
}

/// (inc/transfer.hpp:164-182)
inline HDGVel restrict_advection(const HDGVel& wf, const Space& Vc, const RefineMaps& maps) {
  const Mesh& cm = *Vc.mesh;
  const Mesh& fm = *wf.V.mesh;
  HDGVel wc = HDGVel::zero(Vc);
  for (int cf = 0; cf < cm.nf(); ++cf) {
    V2 nc = cm.fnormal(cf);
    Real flux = 0, tang = 0;
    for (int ff : maps.facet_children[cf]) {
      Real s = nc.dot(fm.fnormal(ff)) > 0 ? 0.5 : -0.5;
      flux += s * wf.compound[wf.V.flux(ff, 0)];
      tang += s * wf.compound[wf.V.tang(ff, 0)];
    }
    wc.compound[Vc.flux(cf, 0)] = flux;
    wc.compound[Vc.tang(cf, 0)] = tang;
  }
  return wc;
}

/// (inc/transfer.hpp:186-195)
inline HDGVel lowest_order_advection(const HDGVel& wk, const Space& V0) {
  HDGVel w0 = HDGVel::zero(V0);
  for (int f = 0; f < V0.mesh->nf(); ++f) {
    w0.compound[V0.flux(f, 0)] = wk.compound[wk.V.flux(f, 0)];
    w0.compound[V0.tang(f, 0)] = wk.compound[wk.V.tang(f, 0)];
  }
  return w0;
}

// ------------------------------------------------------------- smoother ----
/// Free DOFs per vertex patch, (flux_i, tang_i) per facet, empty patches
/// dropped (inc/smoother.hpp:13-28).
inline std::vector<std::vector<Index>> velocity_patches(const Space& V, const Constraints& con) {
  std::vector<std::vector<Index>> out;
  for (const auto& facets : vertex_patches(*V.mesh)) {
    std::vector<Index> d;
    for (int f : facets)
      for (int i = 0; i <= V.k; ++i) {
        Index dn = con.full_to_free[V.flux(f, i)];
        if (dn < 0) continue;
        d.push_back(dn);
        d.push_back(con.full_to_free[V.tang(f, i)]);
      }
    if (!d.empty()) out.push_back(std::move(d));
  }
  return out;
}

/// Overlapping vertex-patch smoother with exact dense patch solves
/// (inc/smoother.hpp:35-100). A^T is held as a CSR of the transpose so that
/// "column i of A" reads as row i of AT.
/// Diagnostic arithmetic variants (env ORC_VARIANT, a bit mask; default 0 =
/// the reference's arithmetic): 1 patch solves by explicit inverses, 2 the
/// coarse solve by an explicit inverse, 4 "pull" sweeps (each patch recomputes
/// its residual rows b_p - A_p x from the current iterate instead of updating
/// a running residual). All are exact-arithmetic identities; they exist to
/// attribute device-vs-reference differences (tools/variant_floor.py).
inline int variant() {
  static const int v = [] {
    const char* e = std::getenv("ORC_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

class PatchSmoother {
 public:
  PatchSmoother(const Csr& A, const Csr& AT, std::vector<std::vector<Index>> patches)
      : a_(&A), at_(&AT), patches_(std::move(patches)) {
    lu_.reserve(patches_.size());
    for (const auto& p : patches_) {
      const int np = int(p.size());
      Mat App(np, np);
      for (int r = 0; r < np; ++r)
        for (int c = 0; c < np; ++c) App(r, c) = a_->coeff(p[r], p[c]);
      lu_.emplace_back(App);
      if (variant() & 1) lu_.back().make_inverse();
    }
  }
  const std::vector<std::vector<Index>>& patches() const { return patches_; }
  void forward(Vec& x, const Vec& b, int sweeps) const {
    if (variant() & 4) {  // pull: r_p = b_p - A_p x at patch time
      for (int s = 0; s < sweeps; ++s)
        for (std::size_t j = 0; j < patches_.size(); ++j) pull_patch(j, x, b, *a_, false);
      return;
    }
    Vec r = residual(x, b);
    for (int s = 0; s < sweeps; ++s)
      for (std::size_t j = 0; j < patches_.size(); ++j) apply_patch(j, x, r, *at_, false);
  }
  void backward(Vec& x, const Vec& b, int sweeps) const {
    Vec y(x.size(), 0.0);
    Vec r = residual(x, b);
    if (variant() & 4) {  // pull: r_p = r0_p - (A^T)_p y at patch time
      for (int s = 0; s < sweeps; ++s)
        for (std::size_t j = patches_.size(); j-- > 0;) pull_patch(j, y, r, *at_, true);
    } else {
      for (int s = 0; s < sweeps; ++s)
        for (std::size_t j = patches_.size(); j-- > 0;) apply_patch(j, y, r, *a_, true);
    }
    for (std::size_t i = 0; i < x.size(); ++i) x[i] += y[i];
  }
  void jacobi(Vec& x, const Vec& b, int sweeps, Real damping) const {
    for (int s = 0; s < sweeps; ++s) {
      Vec r = residual(x, b);
      for (std::size_t j = 0; j < patches_.size(); ++j) {
        const auto& p = patches_[j];
        Vec rp(p.size());
        for (std::size_t i = 0; i < p.size(); ++i) rp[i] = r[p[i]];
        Vec d = lu_[j].solve(rp);
        for (std::size_t i = 0; i < p.size(); ++i) x[p[i]] += damping * d[i];
      }
    }
  }

 private:
  Vec residual(const Vec& x, const Vec& b) const {
    Vec ax = a_->mul(x);
    Vec r(b.size());
    for (std::size_t i = 0; i < b.size(); ++i) r[i] = b[i] - ax[i];
    return r;
  }
  // cols_of: matrix whose ROW i is column i of the operator applied
  void apply_patch(std::size_t j, Vec& x, Vec& r, const Csr& cols_of, bool transposed) const {
    const auto& p = patches_[j];
    Vec rp(p.size());
    for (std::size_t i = 0; i < p.size(); ++i) rp[i] = r[p[i]];
    Vec d = transposed ? lu_[j].solve_t(rp) : lu_[j].solve(rp);
    for (std::size_t i = 0; i < p.size(); ++i) {
      x[p[i]] += d[i];
      for (Index q = cols_of.ptr[p[i]]; q < cols_of.ptr[p[i] + 1]; ++q) r[cols_of.idx[q]] -= cols_of.val[q] * d[i];
    }
  }
  // rows_of: ROW i gives residual row i as a function of the iterate
  void pull_patch(std::size_t j, Vec& x, const Vec& b, const Csr& rows_of, bool transposed) const {
    const auto& p = patches_[j];
    Vec rp(p.size());
    for (std::size_t i = 0; i < p.size(); ++i) {
      Real s = b[p[i]];
      for (Index q = rows_of.ptr[p[i]]; q < rows_of.ptr[p[i] + 1]; ++q) s -= rows_of.val[q] * x[rows_of.idx[q]];
      rp[i] = s;
    }
    Vec d = transposed ? lu_[j].solve_t(rp) : lu_[j].solve(rp);
    for (std::size_t i = 0; i < p.size(); ++i) x[p[i]] += d[i];
  }
  const Csr* a_;
  const Csr* at_;
  std::vector<std::vector<Index>> patches_;
  std::vector<LU> lu_;
};

// ------------------------------------------------------------ multigrid ----
enum Cycle { kV = 0, kW = 1, kVariableV = 2 };
enum SmootherKind { kMultiplicative = 0, kAdditive = 1 };

struct MGOpt {
  int cycle = kW, smoother = kMultiplicative, smooth_steps = 1;
  Real jacobi_damping = 1.0 / 3.0;
};

/// hp-multigrid preconditioner (inc/multigrid.hpp:43-197).
class MG {
 public:
  MG(const Hierarchy& hier, int k, const Field& bc, const AsmOpt& fine, Real inv_eps, const MGOpt& mg)
      : k_(k), mg_(mg), q_(mg.cycle == kW ? 2 : 1), inv_eps_(inv_eps) {
    const int L = int(hier.levels.size()) - 1;
    advected_ = fine.advection != nullptr;
    h_.resize(L + 1);
    for (int l = 0; l <= L; ++l) {
      h_[l].V = Space(hier.levels[l], 0);
      h_[l].con = Constraints::build(h_[l].V, bc);
      h_[l].steps = mg.cycle == kVariableV ? mg.smooth_steps << (L - l) : mg.smooth_steps;
    }
    std::vector<HDGVel> adv;
    if (advected_) {
      adv.resize(L + 1);
      adv[L] = k > 0 ? lowest_order_advection(*fine.advection, h_[L].V) : *fine.advection;
      for (int l = L; l > 0; --l) adv[l - 1] = restrict_advection(adv[l], h_[l - 1].V, hier.maps[l - 1]);
    }
    for (int l = 0; l <= L; ++l) {
      AsmOpt opt;
      opt.nu = fine.nu;
      opt.beta = fine.beta;
      opt.mass_coef = fine.mass_coef;
      opt.newton = fine.newton;
      if (advected_) opt.advection = &adv[l];
      const bool finest = k == 0 && l == L;
      if (finest) {
        opt.load = fine.load;
        opt.elem_load = fine.elem_load;
        opt.mass_field = fine.mass_field;
      }
      Condensed sys = assemble_condensed(hier.levels[l], h_[l].V, h_[l].con, opt);
      Vec drhs;
      Csr D = grad_div(h_[l].V, h_[l].con, h_[l].con.g_full, finest ? &drhs : nullptr);
      h_[l].A = sys.A.add(D, inv_eps);
      h_[l].AT = advected_ ? h_[l].A.transpose() : h_[l].A;
      if (finest) {
        rhs_ = sys.rhs;
        for (std::size_t i = 0; i < rhs_.size(); ++i) rhs_[i] += inv_eps * drhs[i];
      }
    }
    coarse_ = LU(h_[0].A.dense());
    if (variant() & 2) coarse_.make_inverse();
    for (int l = 1; l <= L; ++l) {
      Csr avg = averaging_transfer(h_[l - 1].V, h_[l - 1].con, h_[l].V, h_[l].con, hier.maps[l - 1]);
      h_[l].P = corrected_prolongation(avg, h_[l].A, interior_patch_dofs(h_[l].V, h_[l].con, hier.maps[l - 1]));
      h_[l].PT = h_[l].P.transpose();
      h_[l].sm = std::make_unique<PatchSmoother>(h_[l].A, h_[l].AT, velocity_patches(h_[l].V, h_[l].con));
    }
    if (k_ > 0) {
      head_.V = Space(hier.levels[L], k);
      head_.con = Constraints::build(head_.V, bc);
      head_.steps = mg.smooth_steps;
      Condensed sys = assemble_condensed(hier.levels[L], head_.V, head_.con, fine);
      Vec drhs;
      Csr D = grad_div(head_.V, head_.con, head_.con.g_full, &drhs);
      head_.A = sys.A.add(D, inv_eps);
      head_.AT = advected_ ? head_.A.transpose() : head_.A;
      rhs_ = sys.rhs;
      for (std::size_t i = 0; i < rhs_.size(); ++i) rhs_[i] += inv_eps * drhs[i];
      head_.sm = std::make_unique<PatchSmoother>(head_.A, head_.AT, velocity_patches(head_.V, head_.con));
      E_ = order_embedding(h_[L].V, h_[L].con, head_.V, head_.con);
      ET_ = E_.transpose();
    }
  }
  Vec apply(const Vec& b) const {
    if (k_ == 0) return h_cycle(int(h_.size()) - 1, b);
    Vec x(b.size(), 0.0);
    smooth(head_, x, b, false);
    Vec ax = head_.A.mul(x);
    Vec r(b.size());
    for (std::size_t i = 0; i < b.size(); ++i) r[i] = b[i] - ax[i];
    Vec e = E_.mul(h_cycle(int(h_.size()) - 1, ET_.mul(r)));
    for (std::size_t i = 0; i < b.size(); ++i) x[i] += e[i];
    smooth(head_, x, b, true);
    return x;
  }
  const Csr& matrix() const { return k_ == 0 ? h_.back().A : head_.A; }
  const Space& space() const { return k_ == 0 ? h_.back().V : head_.V; }
  const Constraints& constraints() const { return k_ == 0 ? h_.back().con : head_.con; }
  const Vec& rhs() const { return rhs_; }
  bool symmetric() const { return !advected_; }
  Real penalty() const { return inv_eps_; }
  int levels() const { return int(h_.size()); }
  // introspection for parity tests
  const Csr& level_matrix(int l) const { return h_[l].A; }
  const Csr& level_P(int l) const { return h_[l].P; }
  const Constraints& level_con(int l) const { return h_[l].con; }
  const PatchSmoother* smoother(int l) const { return l < 0 ? head_.sm.get() : h_[l].sm.get(); }

 private:
  struct Level {
    Space V;
    Constraints con;
    Csr A, AT, P, PT;
    std::unique_ptr<PatchSmoother> sm;
    int steps = 1;
  };
  void smooth(const Level& lv, Vec& x, const Vec& b, bool post) const {
    if (mg_.smoother == kAdditive) lv.sm->jacobi(x, b, lv.steps, mg_.jacobi_damping);
    else if (post) lv.sm->backward(x, b, lv.steps);
    else lv.sm->forward(x, b, lv.steps);
  }
  Vec h_cycle(int l, const Vec& b) const {
    if (l == 0) return coarse_.solve(b);
    const Level& lv = h_[l];
    Vec x(b.size(), 0.0);
    smooth(lv, x, b, false);
    Vec ax = lv.A.mul(x);
    Vec r(b.size());
    for (std::size_t i = 0; i < b.size(); ++i) r[i] = b[i] - ax[i];
    Vec rc = lv.PT.mul(r);
    Vec e = h_cycle(l - 1, rc);
    for (int i = 1; i < q_; ++i) {
      Vec ae = h_[l - 1].A.mul(e);
      Vec rr(rc.size());
      for (std::size_t j = 0; j < rc.size(); ++j) rr[j] = rc[j] - ae[j];
      Vec e2 = h_cycle(l - 1, rr);
      for (std::size_t j = 0; j < rc.size(); ++j) e[j] += e2[j];
    }
    Vec pe = lv.P.mul(e);
    for (std::size_t i = 0; i < x.size(); ++i) x[i] += pe[i];
    smooth(lv, x, b, true);
    return x;
  }
  int k_;
  MGOpt mg_;
  int q_;
  Real inv_eps_;
  bool advected_ = false;
  std::vector<Level> h_;
  Level head_;
  LU coarse_;
  Csr E_, ET_;
  Vec rhs_;
};

// --------------------------------------------------------------- krylov ----
using Op = std::function<Vec(const Vec&)>;
struct KrylovOpt {
  Real rel_tol = 1e-8, abs_tol = 1e-10;
  int max_iterations = 500;
  /// GMRES(m) cycle length (BASELINE config 5's restarted GMRes(50)); 0 =
  /// the reference's unrestarted method (krylov.hpp:79-84). An extension of
  /// the reference: a cycle that reaches m Arnoldi steps forms its update
  /// and restarts from the true residual exactly like a recurrence-converged
  /// cycle that failed the true-residual check (krylov.hpp:127-143).
  int restart = 0;
};
struct SolveStats {
  int iterations = 0;
  bool converged = false, not_applicable = false;
  Real residual = 0;
};

/// (inc/krylov.hpp:30-73)
inline SolveStats pcg(const Op& A, const Op& M, const Vec& b, Vec& x, const KrylovOpt& o = {}) {
  SolveStats st;
  const Real target = std::max(o.rel_tol * norm(b), o.abs_tol);
  Vec ax = A(x), r(b.size());
  for (std::size_t i = 0; i < b.size(); ++i) r[i] = b[i] - ax[i];
  st.residual = norm(r);
  if (st.residual <= target) { st.converged = true; return st; }
  Vec z = M(r);
  Real rz = dot(r, z);
  if (rz <= 0) { st.not_applicable = true; return st; }
  Vec p = z;
  for (int it = 0; it < o.max_iterations; ++it) {
    Vec ap = A(p);
    Real pap = dot(p, ap);
    if (pap <= 0) { st.not_applicable = true; return st; }
    Real alpha = rz / pap;
    for (std::size_t i = 0; i < x.size(); ++i) { x[i] += alpha * p[i]; r[i] -= alpha * ap[i]; }
    st.iterations = it + 1;
    st.residual = norm(r);
    if (st.residual <= target) { st.converged = true; return st; }
    z = M(r);
    Real rzn = dot(r, z);
    if (rzn <= 0) { st.not_applicable = true; return st; }
    Real beta = rzn / rz;
    for (std::size_t i = 0; i < p.size(); ++i) p[i] = z[i] + beta * p[i];
    rz = rzn;
  }
  return st;
}

/// Right-preconditioned MGS GMRES with Givens rotations (inc/krylov.hpp:79-144).
inline SolveStats gmres(const Op& A, const Op& M, const Vec& b, Vec& x, const KrylovOpt& o = {}) {
  SolveStats st;
  const Real target = std::max(o.rel_tol * norm(b), o.abs_tol);
  const Real breakdown = 1e-14;
  const std::size_t n = b.size();
  while (st.iterations < o.max_iterations) {
    Vec ax = A(x), r(n);
    for (std::size_t i = 0; i < n; ++i) r[i] = b[i] - ax[i];
    st.residual = norm(r);
    if (st.residual <= target) { st.converged = true; return st; }
    const Real beta = st.residual;
    std::vector<Vec> V;
    V.push_back(r);
    for (auto& v : V[0]) v /= beta;
    std::vector<Vec> hc;
    Vec cs, sn, g{beta};
    bool stalled = false;
    const int cap = o.restart > 0 ? o.restart : (1 << 30);
    for (int j = 0; st.iterations < o.max_iterations && j < cap; ++j) {
      Vec w = A(M(V[j]));
      Vec h(j + 2, 0.0);
      for (int i = 0; i <= j; ++i) {
        h[i] = dot(w, V[i]);
        for (std::size_t t = 0; t < n; ++t) w[t] -= h[i] * V[i][t];
      }
      h[j + 1] = norm(w);
      bool happy = h[j + 1] <= breakdown * beta;
      if (!happy) {
        for (auto& v : w) v /= h[j + 1];
        V.push_back(w);
      }
      for (int i = 0; i < j; ++i) {
        Real t = cs[i] * h[i] + sn[i] * h[i + 1];
        h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
        h[i] = t;
      }
      Real rho = std::hypot(h[j], h[j + 1]);
      cs.push_back(h[j] / rho);
      sn.push_back(h[j + 1] / rho);
      h[j] = rho;
      h[j + 1] = 0;
      g.push_back(-sn.back() * g[j]);
      g[j] *= cs.back();
      hc.push_back(h);
      ++st.iterations;
      if (std::abs(g.back()) <= target || happy) {
        stalled = happy && std::abs(g.back()) > target;
        break;
      }
    }
    const int m = int(hc.size());
    Vec y(m);
    for (int i = m - 1; i >= 0; --i) {
      Real s = g[i];
      for (int l = i + 1; l < m; ++l) s -= hc[l][i] * y[l];
      y[i] = s / hc[i][i];
    }
    Vec u(n, 0.0);
    for (int i = 0; i < m; ++i)
      for (std::size_t t = 0; t < n; ++t) u[t] += y[i] * V[i][t];
    Vec mu = M(u);
    for (std::size_t t = 0; t < n; ++t) x[t] += mu[t];
    Vec ax2 = A(x), r2(n);
    for (std::size_t t = 0; t < n; ++t) r2[t] = b[t] - ax2[t];
    st.residual = norm(r2);
    if (st.residual <= target) { st.converged = true; return st; }
    if (stalled) return st;
  }
  return st;
}

// ---------------------------------------------------------------- uzawa ----
struct UzawaOpt {
  int outer_iterations = 2;
  KrylovOpt krylov;
  const Vec* initial_velocity = nullptr;
};
struct UzawaReport {
  std::vector<int> inner_iterations;
  std::vector<Real> divergence_history;
  bool converged = false, not_applicable = false;
  Real final_divergence = 0;
};
struct StokesSolution {
  Vec velocity, pressure;
  UzawaReport report;
};

/// (inc/uzawa.hpp:40-45)
inline SolveStats inner_solve(const MG& B, const Vec& rhs, Vec& x, const KrylovOpt& o) {
  Op A = [&B](const Vec& v) { return B.matrix().mul(v); };
  Op M = [&B](const Vec& v) { return B.apply(v); };
  return B.symmetric() ? pcg(A, M, rhs, x, o) : gmres(A, M, rhs, x, o);
}

/// (inc/uzawa.hpp:51-91)
inline StokesSolution uzawa(const MG& B, const UzawaOpt& o = {}) {
  const Space& V = B.space();
  const Constraints& con = B.constraints();
  const Mesh& mesh = *V.mesh;
  Csr Bdiv = divergence_rows(V);
  Csr BdivT = Bdiv.transpose();
  Vec areas = element_areas(mesh);
  bool enclosed = true;
  for (const auto& f : mesh.fc)
    if (f.tag == kOutflow) enclosed = false;
  StokesSolution sol;
  sol.pressure.assign(mesh.ne(), 0.0);
  Vec u = o.initial_velocity ? con.to_free(*o.initial_velocity) : Vec(con.n_free, 0.0);
  sol.report.converged = true;
  for (int it = 0; it < o.outer_iterations; ++it) {
    Vec rhs = con.to_free(BdivT.mul(sol.pressure));
    for (std::size_t i = 0; i < rhs.size(); ++i) rhs[i] = B.rhs()[i] + rhs[i];
    SolveStats st = inner_solve(B, rhs, u, o.krylov);
    sol.report.inner_iterations.push_back(st.iterations);
    if (st.not_applicable) {
      sol.report.not_applicable = true;
      sol.report.converged = false;
      break;
    }
    sol.report.converged = sol.report.converged && st.converged;
    sol.velocity = con.to_full(u);
    Vec div = Bdiv.mul(sol.velocity);
    Real mx = 0;
    for (int e = 0; e < mesh.ne(); ++e) {
      div[e] /= areas[e];
      sol.pressure[e] -= B.penalty() * div[e];
      mx = std::max(mx, std::abs(div[e]));
    }
    if (enclosed) {
      Real s = dot(areas, sol.pressure), a = 0;
      for (Real v : areas) a += v;
      for (auto& p : sol.pressure) p -= s / a;
    }
    sol.report.divergence_history.push_back(mx);
  }
  if (!sol.report.divergence_history.empty()) sol.report.final_divergence = sol.report.divergence_history.back();
  if (sol.velocity.empty()) sol.velocity = con.to_full(u);
  return sol;
}

}  // namespace orc
