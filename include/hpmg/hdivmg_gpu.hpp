// Drop-in C++ adapter: the reference hdivmg operator interface on top of the
// hpmg C ABI. Compile it inside the reference tree (it includes the
// reference headers, i.e. Eigen); swap
//     hdivmg::MGPreconditioner B(hier, k, bc, opt, inv_eps, mg);
//     auto sol = hdivmg::uzawa_solve(B);
// for
//     hpmg::MGPreconditioner B(hier, k, bc, opt, inv_eps, mg);
//     auto sol = hpmg::uzawa_solve(B);
// Signatures and semantics follow proj/include/hdivmg/multigrid.hpp:43-146,
// krylov.hpp:30-144, uzawa.hpp:23-91, ns.hpp:69-149 and postprocess.hpp:24-188. Setup errors are rethrown as the
// reference's exception types; Krylov breakdown stays in-band.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hdivmg/multigrid.hpp"
#include "hdivmg/ns.hpp"
#include "hdivmg/postprocess.hpp"
#include "hdivmg/uzawa.hpp"
#include "hpmg/capi.h"

namespace hpmg {

using hdivmg::Index;
using hdivmg::Real;
using hdivmg::Vec;
using hdivmg::Vec2;

namespace detail {
inline void check(int rc, const hpmg_ctx* ctx = nullptr) {
  if (rc == HPMG_OK) return;
  std::string msg = ctx ? hpmg_ctx_error(ctx) : hpmg_last_error();
  if (rc == HPMG_ERR_ARG) throw std::invalid_argument(msg);
  if (rc == HPMG_ERR_LOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}
inline void to_std(const Vec& v, std::vector<double>& out) { out.assign(v.data(), v.data() + v.size()); }
inline void field_trampoline(double x, double y, double* out, void* user) {
  const auto& f = *static_cast<const std::function<Vec2(const Vec2&)>*>(user);
  Vec2 v = f(Vec2(x, y));
  out[0] = v.x();
  out[1] = v.y();
}
inline void tensor_trampoline(double x, double y, double* out, void* user) {
  const auto& f = *static_cast<const std::function<hdivmg::Mat2(const Vec2&)>*>(user);
  const hdivmg::Mat2 g = f(Vec2(x, y));
  out[0] = g(0, 0);
  out[1] = g(0, 1);
  out[2] = g(1, 0);
  out[3] = g(1, 1);
}
}  // namespace detail

class MGPreconditioner {
 public:
  MGPreconditioner(const hdivmg::MeshHierarchy& hier, int k, const hdivmg::VelocityBC& bc,
                   const hdivmg::AssemblyOptions& fine_opt, Real inv_eps, const hdivmg::MGOptions& mg)
      : bc_(bc.g), load_(fine_opt.load) {
    const hdivmg::Mesh& base = hier.levels.front();
    for (const auto& v : base.vertices) {
      xy_.push_back(v.x());
      xy_.push_back(v.y());
    }
    for (const auto& e : base.elements)
      for (int i = 0; i < 3; ++i) el_.push_back(e.v[i]);
    for (const auto& f : base.facets)
      if (f.tag == hdivmg::bc::kOutflow) {
        tags_.push_back(f.a);
        tags_.push_back(f.b);
        tags_.push_back(HPMG_TAG_OUTFLOW);
      }
    hpmg_mesh_desc md{base.nv(), xy_.data(), base.ne(), el_.data(), int(tags_.size() / 3), tags_.data(),
                      int(hier.levels.size())};
    hpmg_options o{k, fine_opt.nu, fine_opt.beta, fine_opt.mass_coef, inv_eps,
                   mg.cycle == hdivmg::CycleKind::V ? HPMG_CYCLE_V
                   : mg.cycle == hdivmg::CycleKind::W ? HPMG_CYCLE_W
                                                      : HPMG_CYCLE_VARIABLE_V,
                   mg.smoother == hdivmg::SmootherKind::Multiplicative ? HPMG_SMOOTH_MULTIPLICATIVE
                                                                       : HPMG_SMOOTH_ADDITIVE,
                   mg.smooth_steps, mg.jacobi_damping, HPMG_SWEEP_RECORDS};
    hpmg_problem p{};
    if (bc_) {
      p.bc = &detail::field_trampoline;
      p.bc_user = &bc_;
    }
    if (load_) {
      p.load = &detail::field_trampoline;
      p.load_user = &load_;
    }
    // Advection / pseudo-time states: the compound part is canonical; the
    // interior coefficients are in the generating library's interior basis,
    // which differs from the reference's in the divergence-free bubbles for
    // k >= 2 (use states produced by hpmg_ns_solve / hpmg_interpolate_hdg, or
    // a point field through hpmg_problem.wind, at k >= 2).
    if (fine_opt.advection) {
      detail::to_std(fine_opt.advection->compound, wind_c_);
      detail::to_std(fine_opt.advection->interior, wind_i_);
      p.wind_compound = wind_c_.data();
      p.wind_interior = wind_i_.data();
      p.newton = fine_opt.newton;
    }
    if (fine_opt.mass_field) {
      detail::to_std(fine_opt.mass_field->compound, mass_c_);
      detail::to_std(fine_opt.mass_field->interior, mass_i_);
      p.mass_compound = mass_c_.data();
      p.mass_interior = mass_i_.data();
    }
    hpmg_ctx* c = nullptr;
    detail::check(hpmg_create(&c, &md, &o, &p));
    ctx_.reset(c);
    // host-side space and constraints of the finest system (multigrid.hpp:138-141):
    // bookkeeping only, built exactly as the reference builds them
    space_ = hdivmg::CompoundSpace(hier.levels.back(), k);
    con_ = hdivmg::Constraints::build(space_, bc);
  }
  MGPreconditioner(const MGPreconditioner&) = delete;
  MGPreconditioner& operator=(const MGPreconditioner&) = delete;

  /// One cycle, zero initial guess (multigrid.hpp:117-128).
  Vec apply(const Vec& b) const {
    Vec z(b.size());
    detail::check(hpmg_apply(ctx_.get(), b.data(), z.data(), 0), ctx_.get());
    return z;
  }
  hdivmg::LinearOperator as_operator() const {
    return [this](const Vec& v) { return apply(v); };
  }
  /// matrix() * v on the device (uzawa.hpp:42)
  Vec spmv(const Vec& v) const {
    Vec y(v.size());
    detail::check(hpmg_spmv(ctx_.get(), v.data(), y.data(), 0), ctx_.get());
    return y;
  }
  /// host mirror of the finest operator (multigrid.hpp:133)
  hdivmg::SpMat matrix() const {
    int64_t nnz = 0;
    detail::check(hpmg_matrix_csr(ctx_.get(), -1, &nnz, nullptr, nullptr, nullptr), ctx_.get());
    const int64_t n = hpmg_n(ctx_.get());
    std::vector<int64_t> ptr(n + 1), idx(nnz);
    std::vector<double> val(nnz);
    detail::check(hpmg_matrix_csr(ctx_.get(), -1, &nnz, ptr.data(), idx.data(), val.data()), ctx_.get());
    std::vector<hdivmg::Triplet> t;
    t.reserve(nnz);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q) t.emplace_back(int(i), int(idx[q]), val[q]);
    hdivmg::SpMat A(static_cast<int>(n), static_cast<int>(n));  // not A(int(n), int(n)): most vexing parse
    A.setFromTriplets(t.begin(), t.end());
    return A;
  }
  /// transpose of matrix() for advected operators, matrix() otherwise (multigrid.hpp:136-138)
  hdivmg::SpMat matrix_transpose() const {
    hdivmg::SpMat A = matrix();
    if (symmetric()) return A;
    return hdivmg::SpMat(A.transpose());
  }
  const hdivmg::CompoundSpace& space() const { return space_; }
  const hdivmg::Constraints& constraints() const { return con_; }
  Vec rhs() const {
    Vec r(hpmg_n(ctx_.get()));
    detail::check(hpmg_rhs(ctx_.get(), r.data(), 0), ctx_.get());
    return r;
  }
  bool symmetric() const { return hpmg_symmetric(ctx_.get()) != 0; }
  Real penalty() const { return hpmg_penalty(ctx_.get()); }
  hpmg_ctx* handle() const { return ctx_.get(); }

 private:
  struct Del {
    void operator()(hpmg_ctx* c) const { hpmg_destroy(c); }
  };
  std::function<Vec2(const Vec2&)> bc_, load_;
  hdivmg::CompoundSpace space_;
  hdivmg::Constraints con_;
  std::vector<double> xy_, wind_c_, wind_i_, mass_c_, mass_i_;
  std::vector<int> el_, tags_;
  std::unique_ptr<hpmg_ctx, Del> ctx_;
};

/// The reference's operator-generic solvers (krylov.hpp:30,79), so call sites
/// written against hdivmg::pcg / hdivmg::gmres with LinearOperator arguments
/// recompile unchanged with `using namespace hpmg` or hpmg:: qualification;
/// with B.as_operator() as M every preconditioner application runs on the
/// device (host vectors in and out). The device-resident loops below
/// (pcg(B, b, x), gmres(B, b, x)) keep the whole iteration on the GPU.
inline hdivmg::SolveStats pcg(const hdivmg::LinearOperator& A, const hdivmg::LinearOperator& M, const Vec& b, Vec& x,
                              const hdivmg::KrylovOptions& opt = {}) {
  return hdivmg::pcg(A, M, b, x, opt);
}
inline hdivmg::SolveStats gmres(const hdivmg::LinearOperator& A, const hdivmg::LinearOperator& M, const Vec& b,
                                Vec& x, const hdivmg::KrylovOptions& opt = {}) {
  return hdivmg::gmres(A, M, b, x, opt);
}
/// A LinearOperator of B.matrix() evaluated on the device (uzawa.hpp:42).
inline hdivmg::LinearOperator matrix_operator(const MGPreconditioner& B) {
  return [&B](const Vec& v) { return B.spmv(v); };
}

/// Device PCG with B.matrix() and B.apply (krylov.hpp:30-73).
inline hdivmg::SolveStats pcg(const MGPreconditioner& B, const Vec& b, Vec& x, const hdivmg::KrylovOptions& opt = {}) {
  hpmg_krylov_opts o{opt.rel_tol, opt.abs_tol, opt.max_iterations, 0};
  hpmg_solve_stats st{};
  detail::check(hpmg_pcg(B.handle(), b.data(), x.data(), &o, &st, 0), B.handle());
  hdivmg::SolveStats s;
  s.iterations = st.iterations;
  s.converged = st.converged != 0;
  s.not_applicable = st.not_applicable != 0;
  s.residual = st.residual;
  return s;
}

/// Device right-preconditioned GMRES (krylov.hpp:79-144).
inline hdivmg::SolveStats gmres(const MGPreconditioner& B, const Vec& b, Vec& x,
                                const hdivmg::KrylovOptions& opt = {}) {
  hpmg_krylov_opts o{opt.rel_tol, opt.abs_tol, opt.max_iterations, 0};
  hpmg_solve_stats st{};
  detail::check(hpmg_gmres(B.handle(), b.data(), x.data(), &o, &st, 0), B.handle());
  hdivmg::SolveStats s;
  s.iterations = st.iterations;
  s.converged = st.converged != 0;
  s.not_applicable = st.not_applicable != 0;
  s.residual = st.residual;
  return s;
}

/// Augmented-Lagrangian Uzawa on the device (uzawa.hpp:51-91).
inline hdivmg::StokesSolution uzawa_solve(const MGPreconditioner& B, const hdivmg::UzawaOptions& opt = {}) {
  hpmg_uzawa_opts o{opt.outer_iterations, {opt.krylov.rel_tol, opt.krylov.abs_tol, opt.krylov.max_iterations, 0},
                    opt.initial_velocity ? opt.initial_velocity->data() : nullptr};
  hdivmg::StokesSolution sol;
  sol.velocity.resize(hpmg_n_full(B.handle()));
  sol.pressure.resize(hpmg_ne(B.handle()));
  hpmg_uzawa_report rep{};
  detail::check(hpmg_uzawa(B.handle(), &o, sol.velocity.data(), sol.pressure.data(), &rep), B.handle());
  for (int i = 0; i < rep.n_outer; ++i) {
    sol.report.inner_iterations.push_back(rep.inner_iterations[i]);
    sol.report.divergence_history.push_back(rep.divergence_history[i]);
  }
  sol.report.converged = rep.converged != 0;
  sol.report.not_applicable = rep.not_applicable != 0;
  sol.report.final_divergence = rep.final_divergence;
  return sol;
}

/// Stationary Navier-Stokes driver on the device (ns.hpp:69-149): same
/// arguments and report; velocity.interior / locals are in this library's
/// interior basis (see the MGPreconditioner note).
inline hdivmg::NSSolution navier_stokes_solve(const hdivmg::MeshHierarchy& hier, int k, const hdivmg::VelocityBC& bc,
                                              Real nu, const std::function<Vec2(const Vec2&)>& load, Real inv_eps,
                                              const hdivmg::NSOptions& opt = {}) {
  const hdivmg::Mesh& base = hier.levels.front();
  std::vector<double> xy;
  std::vector<int> el, tags;
  for (const auto& v : base.vertices) {
    xy.push_back(v.x());
    xy.push_back(v.y());
  }
  for (const auto& e : base.elements)
    for (int i = 0; i < 3; ++i) el.push_back(e.v[i]);
  for (const auto& f : base.facets)
    if (f.tag == hdivmg::bc::kOutflow) {
      tags.push_back(f.a);
      tags.push_back(f.b);
      tags.push_back(HPMG_TAG_OUTFLOW);
    }
  hpmg_mesh_desc md{base.nv(), xy.data(), base.ne(), el.data(), int(tags.size() / 3), tags.data(),
                    int(hier.levels.size())};
  const auto& mg = opt.mg;
  hpmg_options o{k, nu, 0.0, 0.0, inv_eps,
                 mg.cycle == hdivmg::CycleKind::V ? HPMG_CYCLE_V
                 : mg.cycle == hdivmg::CycleKind::W ? HPMG_CYCLE_W
                                                    : HPMG_CYCLE_VARIABLE_V,
                 mg.smoother == hdivmg::SmootherKind::Multiplicative ? HPMG_SMOOTH_MULTIPLICATIVE
                                                                     : HPMG_SMOOTH_ADDITIVE,
                 mg.smooth_steps, mg.jacobi_damping, HPMG_SWEEP_RECORDS};
  std::function<Vec2(const Vec2&)> g = bc.g, f = load;
  hpmg_problem p{};
  if (g) {
    p.bc = &detail::field_trampoline;
    p.bc_user = &g;
  }
  if (f) {
    p.load = &detail::field_trampoline;
    p.load_user = &f;
  }
  hpmg_ns_opts no{opt.picard_tol, opt.newton_rel_tol, opt.newton_abs_tol, opt.max_picard, opt.max_newton,
                  opt.pseudo_time_inv,
                  {opt.uzawa.outer_iterations,
                   {opt.uzawa.krylov.rel_tol, opt.uzawa.krylov.abs_tol, opt.uzawa.krylov.max_iterations, 0},
                   nullptr}};
  const hdivmg::Mesh& mesh = hier.levels.back();
  hdivmg::NSSolution out;
  out.velocity.V = hdivmg::CompoundSpace(mesh, k);
  const int ns = (k + 1) * (k + 2) / 2;
  out.velocity.compound = Vec::Zero(out.velocity.V.n_compound());
  out.velocity.interior = Vec::Zero(Index(mesh.ne()) * k * (k + 1));
  out.pressure = Vec::Zero(mesh.ne());
  out.locals.p_ortho = Vec::Zero(Index(mesh.ne()) * (ns - 1));
  std::vector<double> grad(size_t(mesh.ne()) * 4 * ns);
  hpmg_ns_report r{};
  detail::check(hpmg_ns_solve(&md, &o, &p, &no, out.velocity.compound.data(), out.velocity.interior.data(),
                              out.pressure.data(), &r, out.locals.p_ortho.data(), grad.data()));
  out.locals.interior = out.velocity.interior;
  out.locals.grad_coeffs = hdivmg::Mat(4 * ns, mesh.ne());
  for (int e = 0; e < mesh.ne(); ++e)
    for (int q = 0; q < 4 * ns; ++q) out.locals.grad_coeffs(q, e) = grad[size_t(e) * 4 * ns + q];
  out.report.picard_iterations = r.picard_iterations;
  out.report.newton_iterations = r.newton_iterations;
  out.report.picard_inner.assign(r.picard_inner, r.picard_inner + r.n_picard_inner);
  out.report.newton_inner.assign(r.newton_inner, r.newton_inner + r.n_newton_inner);
  out.report.picard_diffs.assign(r.picard_diffs, r.picard_diffs + std::min(r.picard_iterations, 128));
  out.report.newton_diffs.assign(r.newton_diffs, r.newton_diffs + std::min(r.newton_iterations, 64));
  out.report.converged = r.converged != 0;
  out.report.not_applicable = r.not_applicable != 0;
  out.report.final_divergence = r.final_divergence;
  return out;
}

/// postprocess_velocity (postprocess.hpp:29-80) on the device, on B's finest
/// mesh with B's nu; u.interior in this library's interior basis (the
/// MGPreconditioner note), grad_coeffs as recover_locals / navier_stokes_solve
/// return them. Result: coefficients of the orthonormal P^{k+1} basis, column
/// e = x modes then y modes, exactly as the reference's.
inline hdivmg::PostprocessedVelocity postprocess_velocity(const MGPreconditioner& B, const hdivmg::HDGVelocity& u,
                                                         const hdivmg::Mat& grad_coeffs) {
  const int ne = hpmg_ne(B.handle()), k = u.V.k, nh = (k + 2) * (k + 3) / 2;
  hdivmg::PostprocessedVelocity out;
  out.k_hi = k + 1;
  out.coeffs = hdivmg::Mat::Zero(2 * nh, ne);
  detail::check(hpmg_postprocess(B.handle(), u.compound.data(), u.interior.data(), grad_coeffs.data(),
                                 out.coeffs.data()),
                B.handle());
  return out;
}

/// measure_errors (postprocess.hpp:142-188) on the device; the exact fields are
/// tabulated through the callbacks at the degree-16 rule.
inline hdivmg::ErrorNorms measure_errors(const MGPreconditioner& B, const hdivmg::HDGVelocity& u,
                                         const hdivmg::Mat& grad_coeffs, const hdivmg::PostprocessedVelocity& post,
                                         const std::function<Vec2(const Vec2&)>& exact_velocity,
                                         const std::function<hdivmg::Mat2(const Vec2&)>& exact_gradient) {
  double e[4];
  detail::check(hpmg_measure_errors(B.handle(), u.compound.data(), u.interior.data(), grad_coeffs.data(),
                                    post.coeffs.data(), &detail::field_trampoline,
                                    const_cast<std::function<Vec2(const Vec2&)>*>(&exact_velocity),
                                    &detail::tensor_trampoline,
                                    const_cast<std::function<hdivmg::Mat2(const Vec2&)>*>(&exact_gradient), e),
                B.handle());
  hdivmg::ErrorNorms out;
  out.e_u = e[0];
  out.e_L = e[1];
  out.e_ustar = e[2];
  out.div_u = e[3];
  return out;
}

}  // namespace hpmg
