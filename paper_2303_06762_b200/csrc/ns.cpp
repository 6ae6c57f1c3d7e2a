// Stationary Navier-Stokes driver (reference inc/ns.hpp:69-149) on top of the
// C ABI: every linearised step re-linearises one hp-MG preconditioner in place
// around the current velocity (hpmg_update: condensation, patch inverses,
// coarse inverse on the GPU, CR transfer correction on host threads; the
// hierarchy, plans and wave schedules are built once), solves with AL-Uzawa
// warm-started from the previous velocity, and recovers on the device the
// interior RT coefficients the next linearisation needs.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hpmg/capi.h"

namespace {

struct State {
  std::vector<double> compound, interior, pressure, p_ortho, grad;
};

struct Step {
  hpmg_ctx* ctx = nullptr;
  ~Step() { hpmg_destroy(ctx); }
};

[[noreturn]] void fail(hpmg_ctx* ctx) {
  throw std::runtime_error(ctx ? hpmg_ctx_error(ctx) : hpmg_last_error());
}

}  // namespace

extern "C" int hpmg_ns_solve(const hpmg_mesh_desc* mesh, const hpmg_options* opt_in, const hpmg_problem* prob_in,
                             const hpmg_ns_opts* ns, double* velocity, double* interior, double* pressure,
                             hpmg_ns_report* rep, double* p_ortho, double* grad) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  std::memset(rep, 0, sizeof(*rep));
  try {
    hpmg_options aopt = *opt_in;  // AssemblyOptions{nu, load}: no mass term outside the pseudo-time phase
    aopt.beta = 0.0;
    aopt.mass_coef = 0.0;
    hpmg_problem base{};
    if (prob_in) base = *prob_in;
    base.wind_compound = base.wind_interior = nullptr;
    base.wind = nullptr;
    base.wind_user = nullptr;
    base.mass_compound = base.mass_interior = nullptr;
    base.newton = 0;

    State cur, prev;
    double setup_s = 0.0;
    // the Stokes context (also used for the norms) and one advected context,
    // created for the first Picard step and re-linearised in place afterwards
    // (the reference rebuilds the preconditioner per step, ns.hpp:84)
    Step stokes, adv;
    // one linearised step (ns.hpp:81-100); false on breakdown / non-convergence
    auto linear_step = [&](const hpmg_options& o, const hpmg_problem& p, const State* warm, int* inner, int* ninner,
                           int cap) -> bool {
      const bool advected = p.wind_compound != nullptr;
      Step& st = advected ? adv : stokes;
      const auto ts = clk::now();
      if (!st.ctx) {
        if (hpmg_create(&st.ctx, mesh, &o, &p)) fail(nullptr);
      } else if (hpmg_update(st.ctx, &o, &p)) {
        fail(st.ctx);
      }
      setup_s += std::chrono::duration<double>(clk::now() - ts).count();
      const int64_t nfull = hpmg_n_full(st.ctx);
      const int ne = hpmg_ne(st.ctx);
      hpmg_uzawa_opts uo = ns->uzawa;
      uo.initial_velocity = warm ? warm->compound.data() : nullptr;
      std::vector<double> u(nfull), pr(ne);
      hpmg_uzawa_report ur;
      if (hpmg_uzawa(st.ctx, &uo, u.data(), pr.data(), &ur)) fail(st.ctx);
      for (int i = 0; i < ur.n_outer; ++i)
        if (ninner && *ninner < cap) inner[(*ninner)++] = ur.inner_iterations[i];
      if (ur.not_applicable || !ur.converged) {
        rep->not_applicable = ur.not_applicable;
        return false;
      }
      const int k = o.k, ns_ = (k + 1) * (k + 2) / 2;
      std::vector<double> in(size_t(ne) * k * (k + 1) + 1), po(size_t(ne) * std::max(ns_ - 1, 1) + 1),
          gr(size_t(ne) * 4 * ns_);
      if (hpmg_recover(st.ctx, u.data(), in.data(), po.data(), gr.data())) fail(st.ctx);
      in.resize(size_t(ne) * k * (k + 1));
      po.resize(size_t(ne) * (ns_ - 1));
      cur.compound = std::move(u);
      cur.interior = std::move(in);
      cur.pressure = std::move(pr);
      cur.p_ortho = std::move(po);
      cur.grad = std::move(gr);
      rep->final_divergence = ur.final_divergence;
      return true;
    };
    // ||a - b||_L2 and ||a||_L2 of RT fields (assembly.hpp:487-501), on the device
    auto rt_norm = [&](const std::vector<double>& c, const std::vector<double>& i) {
      const double v = hpmg_rt_l2_norm(stokes.ctx, c.data(), i.data());
      if (v < 0) fail(stokes.ctx);
      return v;
    };
    auto diff = [&](const State& a, const State& b) {
      std::vector<double> dc(a.compound.size()), di(a.interior.size());
      for (size_t i = 0; i < dc.size(); ++i) dc[i] = a.compound[i] - b.compound[i];
      for (size_t i = 0; i < di.size(); ++i) di[i] = a.interior[i] - b.interior[i];
      return rt_norm(dc, di);
    };
    auto finish = [&](int rc) {
      if (!cur.compound.empty()) {
        std::memcpy(velocity, cur.compound.data(), sizeof(double) * cur.compound.size());
        if (!cur.interior.empty()) std::memcpy(interior, cur.interior.data(), sizeof(double) * cur.interior.size());
        std::memcpy(pressure, cur.pressure.data(), sizeof(double) * cur.pressure.size());
        if (p_ortho && !cur.p_ortho.empty()) std::memcpy(p_ortho, cur.p_ortho.data(), sizeof(double) * cur.p_ortho.size());
        if (grad) std::memcpy(grad, cur.grad.data(), sizeof(double) * cur.grad.size());
      }
      rep->setup_seconds = setup_s;
      rep->seconds = std::chrono::duration<double>(clk::now() - t0).count();
      return rc;
    };

    // Stokes initial guess (ns.hpp:102-104)
    int stokes_inner[64], nstokes = 0;
    if (!linear_step(aopt, base, nullptr, stokes_inner, &nstokes, 64)) return finish(0);
    prev = cur;
    // Picard (ns.hpp:106-123)
    double last_picard_diff = 0.0;
    for (int n = 0; n < ns->max_picard; ++n) {
      hpmg_options o = aopt;
      hpmg_problem p = base;
      p.wind_compound = prev.compound.data();
      p.wind_interior = prev.interior.empty() ? nullptr : prev.interior.data();
      if (ns->pseudo_time_inv > 0) {
        o.mass_coef = ns->pseudo_time_inv;
        p.mass_compound = prev.compound.data();
        p.mass_interior = p.wind_interior;
      }
      if (!linear_step(o, p, &prev, rep->picard_inner, &rep->n_picard_inner, 512)) return finish(0);
      ++rep->picard_iterations;
      const double d = diff(cur, prev);
      if (n < 128) rep->picard_diffs[n] = d;
      last_picard_diff = d;
      prev = cur;
      if (d < ns->picard_tol) break;
    }
    if (ns->max_newton == 0) {
      // the last step's difference (picard_diffs keeps only the first 128)
      rep->converged = rep->picard_iterations > 0 && last_picard_diff < ns->picard_tol;
      return finish(0);
    }
    // Newton (ns.hpp:130-147)
    for (int n = 0; n < ns->max_newton; ++n) {
      hpmg_problem p = base;
      p.wind_compound = prev.compound.data();
      p.wind_interior = prev.interior.empty() ? nullptr : prev.interior.data();
      p.newton = 1;
      if (!linear_step(aopt, p, &prev, rep->newton_inner, &rep->n_newton_inner, 256)) return finish(0);
      ++rep->newton_iterations;
      const double d = diff(cur, prev);
      if (n < 64) rep->newton_diffs[n] = d;
      prev = cur;
      const double scale = rt_norm(prev.compound, prev.interior);
      if (d < std::max(ns->newton_rel_tol * scale, ns->newton_abs_tol)) {
        rep->converged = 1;
        break;
      }
    }
    return finish(0);
  } catch (const std::exception& e) {
    rep->seconds = std::chrono::duration<double>(clk::now() - t0).count();
    hpmg_set_last_error(e.what());
    return -1;
  }
}
