// TEST INFRASTRUCTURE ONLY. The real reference: this translation unit
// includes the UNMODIFIED reference headers from
// /root/reference/proj/include/hdivmg (compiled against the Eigen-API shim in
// oracle/eigen_shim, Eigen 3 being absent from the image) and exports the
// same extern "C" surface as the restatement's orc_capi.cpp, so the tests can
// run the reference itself, the restatement and the device library on the
// same seeded inputs. Built by oracle/Makefile into oracle/_ref/libref.so
// only where /root/reference exists (this container); nothing on the GPU box
// needs it. Problem description, BC / load / wind kinds: orc_capi.cpp.
#include <chrono>
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "hdivmg/manufactured.hpp"
#include "hdivmg/multigrid.hpp"
#include "hdivmg/ns.hpp"
#include "hdivmg/postprocess.hpp"
#include "hdivmg/uzawa.hpp"

using namespace hdivmg;
using Field = std::function<Vec2(const Vec2&)>;

extern "C" {
typedef struct {
  int mesh_kind, base_n, levels, k;
  double nu, beta, mass_coef, inv_eps;
  int bc_kind, load_kind;
  const double* load;
  int wind_kind;
  int cycle, smoother, smooth_steps;
  double jacobi_damping;
  int newton, mass_field;
} orc_problem;

typedef struct {
  int iterations, converged, not_applicable;
  double residual;
} orc_stats;

typedef struct {
  double picard_tol, newton_rel_tol, newton_abs_tol;
  int max_picard, max_newton;
  double pseudo_time_inv;
  int outer_iterations;
  double rel_tol, abs_tol;
  int max_iterations;
} orc_ns_opts;

typedef struct {
  int picard_iterations, newton_iterations, n_picard_inner, n_newton_inner;
  int picard_inner[512], newton_inner[256];
  double picard_diffs[128], newton_diffs[64];
  int converged, not_applicable;
  double final_divergence, seconds;
} orc_ns_report;
}

namespace {

Field make_bc(int kind) {
  switch (kind) {
    case 0: return nullptr;
    case 1: return [](const Vec2& x) { return x.y() > 1.0 - 1e-12 ? Vec2(4 * x.x() * (1 - x.x()), 0.0) : Vec2(0, 0); };
    case 2: return [](const Vec2& x) { return Vec2(4 * x.x() * (1 - x.x()), 0.0); };
    case 3: return [](const Vec2& x) { return x.x() < 1e-12 ? Vec2(16 * (1 - x.y()) * (x.y() - 0.5), 0.0) : Vec2(0, 0); };
    case 4: return [](const Vec2& x) { return x.y() > 1.0 - 1e-12 ? Vec2(1.0, 0.0) : Vec2(0, 0); };
    case 5: return [](const Vec2&) { return Vec2(0.8, -0.55); };
    case 6: return [](const Vec2&) { return Vec2(0.0, 0.0); };
  }
  throw std::invalid_argument("bc kind (reference driver)");
}

Field make_named_load(int kind, Real nu, Real beta) {
  switch (kind) {
    case 0: return nullptr;
    case 6: return manufactured::stokes_load(nu, beta);
    case 7: return manufactured::navier_stokes_load(nu);
    case 2: return [](const Vec2& x) { return Vec2(std::sin(2 * x.x()) + x.y(), std::cos(x.y()) - x.x() * x.x()); };
    case 3: return [](const Vec2& x) { return Vec2(std::sin(2 * x.x()), x.y()); };
    case 4: return [](const Vec2& x) { return Vec2(std::sin(3 * x.x()) - x.y(), std::cos(2 * x.y()) + x.x() * x.y()); };
    case 5: return [](const Vec2& x) { return Vec2(std::sin(3 * x.x()) + x.y(), std::cos(2 * x.y()) - x.x() * x.x()); };
  }
  throw std::invalid_argument("load kind (reference driver)");
}

Field make_wind(int kind) {
  switch (kind) {
    case 1: return [](const Vec2& x) { return Vec2(x.y() - 0.5, 0.5 - x.x()); };
    case 2: return [](const Vec2& x) {
      const Real s = std::sin(M_PI * x.x()), t = std::sin(M_PI * x.y());
      return Vec2(M_PI * s * s * std::sin(2 * M_PI * x.y()), -M_PI * std::sin(2 * M_PI * x.x()) * t * t);
    };
  }
  throw std::invalid_argument("wind kind (reference driver)");
}

Vec2 structured_load(const double* F, int n, const Vec2& x) {
  int i = std::min(n - 1, std::max(0, int(std::floor(x.x() * n))));
  int j = std::min(n - 1, std::max(0, int(std::floor(x.y() * n))));
  bool lower = (x.x() - Real(i) / n) >= (x.y() - Real(j) / n);
  std::size_t s = (std::size_t(j) * n + i) * 2 + (lower ? 0 : 1);
  return Vec2(F[2 * s], F[2 * s + 1]);
}

struct Problem {
  MeshHierarchy hier;
  HDGVelocity wind;
  std::vector<double> loadcopy;
  AssemblyOptions opt;
  VelocityBC bc;
  std::unique_ptr<MGPreconditioner> mg;
  std::vector<MGTraceEntry> trace;
  Real setup_seconds = 0;
};

thread_local std::string g_err;

Field problem_load(const orc_problem* p, std::vector<double>& copy) {
  if (p->load_kind == 1) {
    int nf = p->base_n << (p->levels - 1);
    copy.assign(p->load, p->load + std::size_t(4) * nf * nf);
    const double* F = copy.data();
    return [F, nf](const Vec2& x) { return structured_load(F, nf, x); };
  }
  return make_named_load(p->load_kind, p->nu, p->beta);
}

MGOptions mg_options(const orc_problem* p) {
  MGOptions mo;
  mo.cycle = p->cycle == 0 ? CycleKind::V : p->cycle == 1 ? CycleKind::W : CycleKind::VariableV;
  mo.smoother = p->smoother == 0 ? SmootherKind::Multiplicative : SmootherKind::Additive;
  mo.smooth_steps = p->smooth_steps;
  mo.jacobi_damping = p->jacobi_damping;
  return mo;
}

Vec to_vec(const double* x, Index n) {
  Vec v(n);
  std::memcpy(v.data(), x, sizeof(double) * std::size_t(n));
  return v;
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
int orc_is_reference() { return 1; }

void orc_seeded_load(int n, unsigned seed, double lo, double hi, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (std::size_t i = 0; i < std::size_t(4) * n * n; ++i) out[i] = dist(rng);
}

void orc_random_vec(long long n, unsigned seed, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (long long i = 0; i < n; ++i) out[i] = dist(rng);
}

/// MGPreconditioner(hier, k, bc, opt, inv_eps, mg) (inc/multigrid.hpp:45-115);
/// `traced` sets MGOptions::trace (multigrid.hpp:33) to the problem's log.
static void* create(const orc_problem* p, bool traced) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    auto pr = std::make_unique<Problem>();
    pr->hier = MeshHierarchy::build(p->mesh_kind == 0 ? unit_square_mesh(p->base_n) : step_mesh(p->base_n),
                                    p->levels);
    const Mesh& fine = pr->hier.levels.back();
    pr->opt.nu = p->nu;
    pr->opt.beta = p->beta;
    pr->opt.mass_coef = p->mass_coef;
    pr->opt.load = problem_load(p, pr->loadcopy);
    if (p->wind_kind) {
      pr->wind = interpolate_hdg(fine, p->k, make_wind(p->wind_kind));
      pr->opt.advection = &pr->wind;
      pr->opt.newton = p->newton != 0;
      if (p->mass_field) pr->opt.mass_field = &pr->wind;
    }
    pr->bc.g = make_bc(p->bc_kind);
    MGOptions mo = mg_options(p);
    if (traced) mo.trace = &pr->trace;
    pr->mg = std::make_unique<MGPreconditioner>(pr->hier, p->k, pr->bc, pr->opt, p->inv_eps, mo);
    pr->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return pr.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* orc_mg_create(const orc_problem* p) { return create(p, false); }
void* orc_mg_create_traced(const orc_problem* p) { return create(p, true); }

void orc_mg_destroy(void* h) { delete static_cast<Problem*>(h); }
double orc_mg_setup_seconds(void* h) { return static_cast<Problem*>(h)->setup_seconds; }
long long orc_mg_n(void* h) { return static_cast<Problem*>(h)->mg->constraints().n_free; }
long long orc_mg_n_full(void* h) { return static_cast<Problem*>(h)->mg->constraints().n_full; }
int orc_mg_ne(void* h) { return static_cast<Problem*>(h)->mg->space().mesh->ne(); }

void orc_mg_free_to_full(void* h, long long* out) {
  const auto& c = static_cast<Problem*>(h)->mg->constraints();
  for (Index i = 0; i < c.n_free; ++i) out[i] = c.free_to_full[std::size_t(i)];
}
void orc_mg_g_full(void* h, double* out) {
  const auto& c = static_cast<Problem*>(h)->mg->constraints();
  std::memcpy(out, c.g_full.data(), sizeof(double) * std::size_t(c.n_full));
}
void orc_mg_rhs(void* h, double* out) {
  const Vec& r = static_cast<Problem*>(h)->mg->rhs();
  std::memcpy(out, r.data(), sizeof(double) * std::size_t(r.size()));
}

/// matrix() (multigrid.hpp:135) as CSR (the reference stores CSC; the
/// operator is transposed storage-wise, values unchanged). Only level -1
/// (the finest system) is public in the reference.
long long orc_mg_nnz(void* h, int) { return static_cast<Problem*>(h)->mg->matrix().nonZeros(); }
long long orc_mg_rows(void* h, int) { return static_cast<Problem*>(h)->mg->matrix().rows(); }
void orc_mg_csr(void* h, int, long long* ptr, long long* idx, double* val) {
  Eigen::SparseMatrix<Real, Eigen::RowMajor> A(static_cast<Problem*>(h)->mg->matrix());
  const Index n = A.rows();
  for (Index i = 0; i < n; ++i) {
    ptr[i] = 0;
  }
  Index t = 0;
  for (Index i = 0; i < n; ++i) {
    ptr[i] = t;
    for (Eigen::SparseMatrix<Real, Eigen::RowMajor>::InnerIterator it(A, i); it; ++it, ++t) {
      idx[t] = it.col();
      val[t] = it.value();
    }
  }
  ptr[n] = t;
}

void orc_mg_spmv(void* h, const double* x, double* y) {
  const SpMat& A = static_cast<Problem*>(h)->mg->matrix();
  Vec yv = A * to_vec(x, A.cols());
  std::memcpy(y, yv.data(), sizeof(double) * std::size_t(A.rows()));
}

/// MGPreconditioner::apply (multigrid.hpp:117-128).
void orc_mg_apply(void* h, const double* b, double* x) {
  auto* p = static_cast<Problem*>(h);
  const Index n = p->mg->constraints().n_free;
  Vec xv = p->mg->apply(to_vec(b, n));
  std::memcpy(x, xv.data(), sizeof(double) * std::size_t(n));
}

/// MG residual trace (MGTraceEntry, multigrid.hpp:18-33,120,126,168-183) of
/// the last apply() of a context made by orc_mg_create_traced: writes up to
/// `cap` (level, entering, residual) triples, returns the number recorded.
int orc_mg_trace(void* h, int cap, int* level, int* entering, double* residual) {
  auto* p = static_cast<Problem*>(h);
  const int n = int(p->trace.size());
  for (int i = 0; i < n && i < cap; ++i) {
    level[i] = p->trace[std::size_t(i)].level;
    entering[i] = p->trace[std::size_t(i)].entering;
    residual[i] = p->trace[std::size_t(i)].residual;
  }
  p->trace.clear();
  return n;
}

/// velocity_patches (smoother.hpp:13-28) of the finest system.
int orc_mg_num_patches(void* h, int) {
  auto* p = static_cast<Problem*>(h);
  return int(velocity_patches(p->mg->space(), p->mg->constraints()).size());
}
long long orc_mg_patches(void* h, int, long long* offs, long long* dofs) {
  auto* p = static_cast<Problem*>(h);
  const auto P = velocity_patches(p->mg->space(), p->mg->constraints());
  long long t = 0;
  for (std::size_t j = 0; j < P.size(); ++j) {
    if (offs) offs[j] = t;
    for (int d : P[j]) {
      if (dofs) dofs[t] = d;
      ++t;
    }
  }
  if (offs) offs[P.size()] = t;
  return t;
}

/// pcg / gmres (krylov.hpp:30-144) with A = matrix(), M = apply, as
/// inner_solve (uzawa.hpp:40-45) wires them.
void orc_mg_krylov(void* h, int method, const double* b, double* x, double rel_tol, double abs_tol, int max_it,
                   orc_stats* out) {
  auto* p = static_cast<Problem*>(h);
  const Index n = p->mg->constraints().n_free;
  Vec bv = to_vec(b, n), xv = to_vec(x, n);
  KrylovOptions o;
  o.rel_tol = rel_tol;
  o.abs_tol = abs_tol;
  o.max_iterations = max_it;
  const MGPreconditioner& B = *p->mg;
  LinearOperator A = [&B](const Vec& v) { return Vec(B.matrix() * v); };
  SolveStats st = method == 0 ? pcg(A, B.as_operator(), bv, xv, o) : gmres(A, B.as_operator(), bv, xv, o);
  std::memcpy(x, xv.data(), sizeof(double) * std::size_t(n));
  out->iterations = st.iterations;
  out->converged = st.converged;
  out->not_applicable = st.not_applicable;
  out->residual = st.residual;
}

/// uzawa_solve (uzawa.hpp:51-91).
int orc_mg_uzawa(void* h, int outer, double rel_tol, double abs_tol, int max_it, double* velocity, double* pressure,
                 int* inner, double* div_hist, int* flags, double* seconds, const double* initial_full) {
  auto* p = static_cast<Problem*>(h);
  UzawaOptions o;
  o.outer_iterations = outer;
  o.krylov.rel_tol = rel_tol;
  o.krylov.abs_tol = abs_tol;
  o.krylov.max_iterations = max_it;
  Vec init;
  if (initial_full) {
    init = to_vec(initial_full, p->mg->constraints().n_full);
    o.initial_velocity = &init;
  }
  auto t0 = std::chrono::steady_clock::now();
  StokesSolution s = uzawa_solve(*p->mg, o);
  if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::memcpy(velocity, s.velocity.data(), sizeof(double) * std::size_t(s.velocity.size()));
  std::memcpy(pressure, s.pressure.data(), sizeof(double) * std::size_t(s.pressure.size()));
  for (std::size_t i = 0; i < s.report.inner_iterations.size(); ++i) inner[i] = s.report.inner_iterations[i];
  for (std::size_t i = 0; i < s.report.divergence_history.size(); ++i) div_hist[i] = s.report.divergence_history[i];
  flags[0] = s.report.converged;
  flags[1] = s.report.not_applicable;
  return int(s.report.inner_iterations.size());
}

/// recover_locals (assembly.hpp:513-549); grad written [ne][4 ns].
void orc_mg_recover(void* h, const double* compound_full, double* interior, double* p_ortho, double* grad) {
  auto* p = static_cast<Problem*>(h);
  const CompoundSpace& V = p->mg->space();
  LocalSolution s = recover_locals(*V.mesh, V, p->opt, to_vec(compound_full, V.n_compound()));
  std::memcpy(interior, s.interior.data(), sizeof(double) * std::size_t(s.interior.size()));
  std::memcpy(p_ortho, s.p_ortho.data(), sizeof(double) * std::size_t(s.p_ortho.size()));
  for (Index e = 0; e < s.grad_coeffs.cols(); ++e)
    for (Index r = 0; r < s.grad_coeffs.rows(); ++r)
      grad[std::size_t(e * s.grad_coeffs.rows() + r)] = s.grad_coeffs(r, e);
}

/// rt_l2_norm (assembly.hpp:487-501) of (compound, interior) on the finest space.
double orc_mg_rt_l2_norm(void* h, const double* compound_full, const double* interior) {
  auto* p = static_cast<Problem*>(h);
  const CompoundSpace& V = p->mg->space();
  return rt_l2_norm(*V.mesh, V, to_vec(compound_full, V.n_compound()), to_vec(interior, V.n_rt_interior()));
}

void orc_mg_wind(void* h, double* compound, double* interior) {
  auto* p = static_cast<Problem*>(h);
  std::memcpy(compound, p->wind.compound.data(), sizeof(double) * std::size_t(p->wind.compound.size()));
  if (p->wind.interior.size())
    std::memcpy(interior, p->wind.interior.data(), sizeof(double) * std::size_t(p->wind.interior.size()));
}

/// Timed setup + Uzawa (time-to-solution, the CPU baseline of bench.py):
/// seconds[0] = MGPreconditioner construction, seconds[1] = uzawa_solve,
/// seconds[2] = recover_locals.
int orc_tts(const orc_problem* p, int outer, double rel_tol, int* inner, double* seconds) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    std::unique_ptr<Problem> pr(static_cast<Problem*>(orc_mg_create(p)));
    if (!pr) return -1;
    auto t1 = std::chrono::steady_clock::now();
    UzawaOptions o;
    o.outer_iterations = outer;
    o.krylov.rel_tol = rel_tol;
    StokesSolution s = uzawa_solve(*pr->mg, o);
    auto t2 = std::chrono::steady_clock::now();
    const CompoundSpace& V = pr->mg->space();
    LocalSolution loc = recover_locals(*V.mesh, V, pr->opt, s.velocity);
    auto t3 = std::chrono::steady_clock::now();
    for (std::size_t i = 0; i < s.report.inner_iterations.size(); ++i) inner[i] = s.report.inner_iterations[i];
    seconds[0] = std::chrono::duration<double>(t1 - t0).count();
    seconds[1] = std::chrono::duration<double>(t2 - t1).count();
    seconds[2] = std::chrono::duration<double>(t3 - t2).count();
    (void)loc;
    return int(s.report.inner_iterations.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

/// navier_stokes_solve (ns.hpp:69-149) of the reference itself, same surface
/// as the restatement's orc_ns_solve (orc_capi.cpp).
int orc_ns_solve(const orc_problem* p, const orc_ns_opts* o, double* velocity, double* interior, double* pressure,
                 orc_ns_report* rep) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    MeshHierarchy hier =
        MeshHierarchy::build(p->mesh_kind == 0 ? unit_square_mesh(p->base_n) : step_mesh(p->base_n), p->levels);
    std::vector<double> loadcopy;
    Field load = problem_load(p, loadcopy);
    NSOptions no;
    no.picard_tol = o->picard_tol;
    no.newton_rel_tol = o->newton_rel_tol;
    no.newton_abs_tol = o->newton_abs_tol;
    no.max_picard = o->max_picard;
    no.max_newton = o->max_newton;
    no.pseudo_time_inv = o->pseudo_time_inv;
    no.mg = mg_options(p);
    no.uzawa.outer_iterations = o->outer_iterations;
    no.uzawa.krylov.rel_tol = o->rel_tol;
    no.uzawa.krylov.abs_tol = o->abs_tol;
    no.uzawa.krylov.max_iterations = o->max_iterations;
    VelocityBC bc;
    bc.g = make_bc(p->bc_kind);
    NSSolution sol = navier_stokes_solve(hier, p->k, bc, p->nu, load, p->inv_eps, no);
    std::memset(rep, 0, sizeof(*rep));
    rep->picard_iterations = sol.report.picard_iterations;
    rep->newton_iterations = sol.report.newton_iterations;
    rep->n_picard_inner = int(std::min<std::size_t>(sol.report.picard_inner.size(), 512));
    rep->n_newton_inner = int(std::min<std::size_t>(sol.report.newton_inner.size(), 256));
    for (int i = 0; i < rep->n_picard_inner; ++i) rep->picard_inner[i] = sol.report.picard_inner[std::size_t(i)];
    for (int i = 0; i < rep->n_newton_inner; ++i) rep->newton_inner[i] = sol.report.newton_inner[std::size_t(i)];
    for (std::size_t i = 0; i < sol.report.picard_diffs.size() && i < 128; ++i)
      rep->picard_diffs[i] = sol.report.picard_diffs[i];
    for (std::size_t i = 0; i < sol.report.newton_diffs.size() && i < 64; ++i)
      rep->newton_diffs[i] = sol.report.newton_diffs[i];
    rep->converged = sol.report.converged;
    rep->not_applicable = sol.report.not_applicable;
    rep->final_divergence = sol.report.final_divergence;
    if (sol.velocity.compound.size()) {
      std::memcpy(velocity, sol.velocity.compound.data(), sizeof(double) * std::size_t(sol.velocity.compound.size()));
      if (sol.velocity.interior.size())
        std::memcpy(interior, sol.velocity.interior.data(), sizeof(double) * std::size_t(sol.velocity.interior.size()));
      std::memcpy(pressure, sol.pressure.data(), sizeof(double) * std::size_t(sol.pressure.size()));
    }
    rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

double orc_mg_time_apply(void* h, int reps) {
  auto* p = static_cast<Problem*>(h);
  const Index n = p->mg->constraints().n_free;
  Vec b(n);
  std::mt19937 rng(47);
  std::uniform_real_distribution<double> d(-1, 1);
  for (Index i = 0; i < n; ++i) b[i] = d(rng);
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    Vec x = p->mg->apply(b);
    b[0] += 1e-300 * x[0];
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"
