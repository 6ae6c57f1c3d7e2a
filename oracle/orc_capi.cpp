// TEST INFRASTRUCTURE ONLY (see orc_core.hpp). extern "C" surface of the
// oracle for the Python test-suite (ctypes) and bench.py's CPU baseline leg.
#include <chrono>
#include <cstring>
#include <random>

#include "orc_mg.hpp"
#include "orc_ns.hpp"
#include "orc_post.hpp"

using namespace orc;

extern "C" {

/// Problem description shared with tests/oracle.py (keep in sync).
typedef struct {
  int mesh_kind;   // 0 unit square, 1 step domain
  int base_n;      // unit_square_mesh(base_n) / step_mesh(base_n)
  int levels;      // MeshHierarchy::build(.., levels)
  int k;
  double nu, beta, mass_coef, inv_eps;
  int bc_kind;     // see make_bc
  int load_kind;   // see make_load
  const double* load;  // load_kind 1: 4 * n_f^2 values, structured (j,i,lower/upper,(fx,fy))
  int wind_kind;   // 0 none, 1 rotation, 2 curl of sin^2(pi x) sin^2(pi y)
  int cycle, smoother, smooth_steps;
  double jacobi_damping;
  int newton;      // Newton linearisation about the wind (AssemblyOptions::newton)
  int mass_field;  // 1: pseudo-time mass field = the interpolated wind (AssemblyOptions::mass_field)
} orc_problem;

typedef struct {
  int iterations, converged, not_applicable;
  double residual;
} orc_stats;

/// NSOptions (inc/ns.hpp:10-28) + the Uzawa/Krylov options of every step.
typedef struct {
  double picard_tol, newton_rel_tol, newton_abs_tol;
  int max_picard, max_newton;
  double pseudo_time_inv;
  int outer_iterations;
  double rel_tol, abs_tol;
  int max_iterations;
} orc_ns_opts;

/// NSReport (inc/ns.hpp:30-53), fixed capacity.
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
    case 1: return [](const V2& x) { return x.y > 1.0 - 1e-12 ? V2(4 * x.x * (1 - x.x), 0.0) : V2(0, 0); };
    case 2: return [](const V2& x) { return V2(4 * x.x * (1 - x.x), 0.0); };
    case 3: return [](const V2& x) { return x.x < 1e-12 ? V2(16 * (1 - x.y) * (x.y - 0.5), 0.0) : V2(0, 0); };
    case 4: return [](const V2& x) { return x.y > 1.0 - 1e-12 ? V2(1.0, 0.0) : V2(0, 0); };
    case 5: return [](const V2&) { return V2(0.8, -0.55); };
    case 6: return [](const V2&) { return V2(0.0, 0.0); };
    case 7: return [](const V2& x) { return linflow::velocity(x); };  // test_postprocess.cpp:138-139
  }
  throw std::invalid_argument("bc kind");
}

Field make_named_load(int kind, Real nu = 0.0, Real beta = 0.0) {
  switch (kind) {
    case 0: return nullptr;
    case 6: return [nu, beta](const V2& x) { return mms::stokes_load(nu, beta, x); };
    case 7: return [nu](const V2& x) { return mms::ns_load(nu, x); };
    case 8: return [](const V2& x) {  // tests/test_postprocess.cpp:133-135
      const V2 u = linflow::velocity(x);
      return V2(2.0 * u.x + 1.0, 2.0 * u.y + 1.0);
    };
    case 2: return [](const V2& x) { return V2(std::sin(2 * x.x) + x.y, std::cos(x.y) - x.x * x.x); };
    case 3: return [](const V2& x) { return V2(std::sin(2 * x.x), x.y); };
    case 4: return [](const V2& x) { return V2(std::sin(3 * x.x) - x.y, std::cos(2 * x.y) + x.x * x.y); };
    case 5: return [](const V2& x) { return V2(std::sin(3 * x.x) + x.y, std::cos(2 * x.y) - x.x * x.x); };
  }
  throw std::invalid_argument("load kind");
}

Field make_wind(int kind) {
  switch (kind) {
    case 1: return [](const V2& x) { return V2(x.y - 0.5, 0.5 - x.x); };
    case 2: return [](const V2& x) {
      const Real s = std::sin(M_PI * x.x), t = std::sin(M_PI * x.y);
      return V2(M_PI * s * s * std::sin(2 * M_PI * x.y), -M_PI * std::sin(2 * M_PI * x.x) * t * t);
    };
  }
  throw std::invalid_argument("wind kind");
}

/// Point location in the structured n x n diagonal mesh of the unit square:
/// cell (i,j), lower triangle (v00,v10,v11) iff (x-i/n) >= (y-j/n)
/// (reference inc/mesh.hpp:231-232).
V2 structured_load(const double* F, int n, const V2& x) {
  int i = std::min(n - 1, std::max(0, int(std::floor(x.x * n))));
  int j = std::min(n - 1, std::max(0, int(std::floor(x.y * n))));
  bool lower = (x.x - Real(i) / n) >= (x.y - Real(j) / n);
  std::size_t s = (std::size_t(j) * n + i) * 2 + (lower ? 0 : 1);
  return V2(F[2 * s], F[2 * s + 1]);
}

struct Problem {
  Hierarchy hier;
  HDGVel wind;
  Vec loadcopy;
  AsmOpt opt;
  std::unique_ptr<MG> mg;
  Real setup_seconds = 0;
  int restart = 0;  // GMRES(m) cycle length for krylov / uzawa calls (0: unrestarted)
};

Mesh base_mesh(const orc_problem* p) {
  return p->mesh_kind == 0 ? unit_square(p->base_n) : step_domain(p->base_n);
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

/// Raise the highest accepted order beyond the reference's 3 (device tests of
/// k = 4..6 only; returns the previous value).
int orc_set_max_order(int k) {
  const int old = max_order();
  max_order() = k;
  return old;
}

/// Seeded per-triangle force: std::mt19937(seed) and
/// std::uniform_real_distribution<double>(lo, hi), drawn in structured
/// (j, i, lower/upper, (fx, fy)) order.
void orc_seeded_load(int n, unsigned seed, double lo, double hi, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (std::size_t i = 0; i < std::size_t(4) * n * n; ++i) out[i] = dist(rng);
}

void* orc_mg_create(const orc_problem* p) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    auto pr = std::make_unique<Problem>();
    pr->hier = Hierarchy::build(base_mesh(p), p->levels);
    const Mesh& fine = pr->hier.levels.back();
    pr->opt.nu = p->nu;
    pr->opt.beta = p->beta;
    pr->opt.mass_coef = p->mass_coef;
    if (p->load_kind == 1) {
      int nf = p->base_n << (p->levels - 1);
      pr->loadcopy.assign(p->load, p->load + std::size_t(4) * nf * nf);
      const double* F = pr->loadcopy.data();
      pr->opt.load = [F, nf](const V2& x) { return structured_load(F, nf, x); };
    } else {
      pr->opt.load = make_named_load(p->load_kind, p->nu, p->beta);
    }
    if (p->wind_kind) {
      pr->wind = interpolate_hdg(fine, p->k, make_wind(p->wind_kind));
      pr->opt.advection = &pr->wind;
      pr->opt.newton = p->newton != 0;
      if (p->mass_field) pr->opt.mass_field = &pr->wind;
    }
    MGOpt mo;
    mo.cycle = p->cycle;
    mo.smoother = p->smoother;
    mo.smooth_steps = p->smooth_steps;
    mo.jacobi_damping = p->jacobi_damping;
    pr->mg = std::make_unique<MG>(pr->hier, p->k, make_bc(p->bc_kind), pr->opt, p->inv_eps, mo);
    pr->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return pr.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void orc_mg_destroy(void* h) { delete static_cast<Problem*>(h); }
/// GMRES(m) cycle length used by the next orc_mg_krylov / orc_mg_uzawa calls.
void orc_mg_set_restart(void* h, int m) { static_cast<Problem*>(h)->restart = m; }
double orc_mg_setup_seconds(void* h) { return static_cast<Problem*>(h)->setup_seconds; }
long long orc_mg_n(void* h) { return static_cast<Problem*>(h)->mg->constraints().n_free; }
long long orc_mg_n_full(void* h) { return static_cast<Problem*>(h)->mg->constraints().n_full; }
int orc_mg_num_levels(void* h) { return static_cast<Problem*>(h)->mg->levels(); }
int orc_mg_ne(void* h) { return static_cast<Problem*>(h)->mg->space().mesh->ne(); }

void orc_mg_free_to_full(void* h, long long* out) {
  const auto& c = static_cast<Problem*>(h)->mg->constraints();
  for (Index i = 0; i < c.n_free; ++i) out[i] = c.free_to_full[i];
}
void orc_mg_g_full(void* h, double* out) {
  const auto& c = static_cast<Problem*>(h)->mg->constraints();
  std::memcpy(out, c.g_full.data(), sizeof(double) * c.n_full);
}
void orc_mg_rhs(void* h, double* out) {
  const auto& r = static_cast<Problem*>(h)->mg->rhs();
  std::memcpy(out, r.data(), sizeof(double) * r.size());
}

/// level: -1 = the finest system operator (head for k>=1), else lowest-order level l.
static const Csr& pick(Problem* p, int level) { return level < 0 ? p->mg->matrix() : p->mg->level_matrix(level); }
long long orc_mg_nnz(void* h, int level) { return pick(static_cast<Problem*>(h), level).nnz(); }
long long orc_mg_rows(void* h, int level) { return pick(static_cast<Problem*>(h), level).rows; }
void orc_mg_csr(void* h, int level, long long* ptr, long long* idx, double* val) {
  const Csr& A = pick(static_cast<Problem*>(h), level);
  for (Index i = 0; i <= A.rows; ++i) ptr[i] = A.ptr[i];
  for (Index p = 0; p < A.nnz(); ++p) { idx[p] = A.idx[p]; val[p] = A.val[p]; }
}
long long orc_mg_P_nnz(void* h, int level) { return static_cast<Problem*>(h)->mg->level_P(level).nnz(); }
void orc_mg_P_csr(void* h, int level, long long* ptr, long long* idx, double* val) {
  const Csr& A = static_cast<Problem*>(h)->mg->level_P(level);
  for (Index i = 0; i <= A.rows; ++i) ptr[i] = A.ptr[i];
  for (Index p = 0; p < A.nnz(); ++p) { idx[p] = A.idx[p]; val[p] = A.val[p]; }
}

void orc_mg_spmv(void* h, const double* x, double* y) {
  const Csr& A = static_cast<Problem*>(h)->mg->matrix();
  Vec xv(x, x + A.rows);
  Vec yv = A.mul(xv);
  std::memcpy(y, yv.data(), sizeof(double) * A.rows);
}

void orc_mg_apply(void* h, const double* b, double* x) {
  auto* p = static_cast<Problem*>(h);
  Index n = p->mg->constraints().n_free;
  Vec bv(b, b + n);
  Vec xv = p->mg->apply(bv);
  std::memcpy(x, xv.data(), sizeof(double) * n);
}

/// Smoother on level l (-1 = head) with sweeps; which: 0 forward, 1 backward, 2 jacobi.
void orc_mg_smooth(void* h, int level, int which, double* x, const double* b, int sweeps, double damping) {
  auto* p = static_cast<Problem*>(h);
  const PatchSmoother* s = p->mg->smoother(level);
  Index n = level < 0 ? p->mg->matrix().rows : p->mg->level_matrix(level).rows;
  Vec xv(x, x + n), bv(b, b + n);
  if (which == 0) s->forward(xv, bv, sweeps);
  else if (which == 1) s->backward(xv, bv, sweeps);
  else s->jacobi(xv, bv, sweeps, damping);
  std::memcpy(x, xv.data(), sizeof(double) * n);
}

int orc_mg_num_patches(void* h, int level) {
  const PatchSmoother* s = static_cast<Problem*>(h)->mg->smoother(level);
  return s ? int(s->patches().size()) : -1;
}
/// Writes patch offsets (np+1) and concatenated DOF lists; returns total size.
long long orc_mg_patches(void* h, int level, long long* offs, long long* dofs) {
  const auto& P = static_cast<Problem*>(h)->mg->smoother(level)->patches();
  long long t = 0;
  for (std::size_t j = 0; j < P.size(); ++j) {
    if (offs) offs[j] = t;
    for (Index d : P[j]) {
      if (dofs) dofs[t] = d;
      ++t;
    }
  }
  if (offs) offs[P.size()] = t;
  return t;
}

void orc_mg_krylov(void* h, int method, const double* b, double* x, double rel_tol, double abs_tol, int max_it,
                   orc_stats* out) {
  auto* p = static_cast<Problem*>(h);
  Index n = p->mg->constraints().n_free;
  Vec bv(b, b + n), xv(x, x + n);
  KrylovOpt o{rel_tol, abs_tol, max_it, p->restart};
  Op A = [p](const Vec& v) { return p->mg->matrix().mul(v); };
  Op M = [p](const Vec& v) { return p->mg->apply(v); };
  SolveStats st = method == 0 ? pcg(A, M, bv, xv, o) : gmres(A, M, bv, xv, o);
  std::memcpy(x, xv.data(), sizeof(double) * n);
  out->iterations = st.iterations;
  out->converged = st.converged;
  out->not_applicable = st.not_applicable;
  out->residual = st.residual;
}

/// Runs uzawa_solve; velocity is full compound (n_full), pressure ne,
/// inner[outer_max] iteration counts; returns number of outer steps done.
int orc_mg_uzawa(void* h, int outer, double rel_tol, double abs_tol, int max_it, double* velocity, double* pressure,
                 int* inner, double* div_hist, int* flags, double* seconds, const double* initial_full) {
  auto* p = static_cast<Problem*>(h);
  UzawaOpt o;
  o.outer_iterations = outer;
  o.krylov = {rel_tol, abs_tol, max_it, p->restart};
  Vec init;
  if (initial_full) {  // warm start (UzawaOptions::initial_velocity)
    init.assign(initial_full, initial_full + p->mg->constraints().n_full);
    o.initial_velocity = &init;
  }
  auto t0 = std::chrono::steady_clock::now();
  StokesSolution s = uzawa(*p->mg, o);
  if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::memcpy(velocity, s.velocity.data(), sizeof(double) * s.velocity.size());
  std::memcpy(pressure, s.pressure.data(), sizeof(double) * s.pressure.size());
  for (std::size_t i = 0; i < s.report.inner_iterations.size(); ++i) inner[i] = s.report.inner_iterations[i];
  for (std::size_t i = 0; i < s.report.divergence_history.size(); ++i) div_hist[i] = s.report.divergence_history[i];
  flags[0] = s.report.converged;
  flags[1] = s.report.not_applicable;
  return int(s.report.inner_iterations.size());
}

/// recover_locals on the finest system for a full compound velocity.
void orc_mg_recover(void* h, const double* compound_full, double* interior, double* p_ortho, double* grad) {
  auto* p = static_cast<Problem*>(h);
  const Space& V = p->mg->space();
  Vec cf(compound_full, compound_full + V.n_compound());
  LocalSolution s = recover_locals(*V.mesh, V, p->opt, cf);
  std::memcpy(interior, s.interior.data(), sizeof(double) * s.interior.size());
  std::memcpy(p_ortho, s.p_ortho.data(), sizeof(double) * s.p_ortho.size());
  // grad: 4ns x ne column-major by element (column e contiguous)
  for (int e = 0; e < s.grad.c; ++e)
    for (int r = 0; r < s.grad.r; ++r) grad[std::size_t(e) * s.grad.r + r] = s.grad(r, e);
}

/// Wind (compound full + interior) interpolated like the problem does.
void orc_mg_wind(void* h, double* compound, double* interior) {
  auto* p = static_cast<Problem*>(h);
  std::memcpy(compound, p->wind.compound.data(), sizeof(double) * p->wind.compound.size());
  if (!p->wind.interior.empty()) std::memcpy(interior, p->wind.interior.data(), sizeof(double) * p->wind.interior.size());
}

/// rt_l2_norm (inc/assembly.hpp:487-501) on the problem's finest space.
double orc_mg_rt_l2_norm(void* h, const double* compound_full, const double* interior) {
  auto* p = static_cast<Problem*>(h);
  const Space& V = p->mg->space();
  Vec c(compound_full, compound_full + V.n_compound());
  Vec i(interior, interior + V.n_interior());
  return rt_l2_norm(*V.mesh, V, c, i);
}

/// postprocess_velocity (inc/postprocess.hpp:29-80): post [ne][2 ns_hi];
/// grad [ne][4 ns] as orc_mg_recover writes it.
void orc_mg_postprocess(void* h, const double* compound_full, const double* interior, const double* grad, double* post) {
  auto* p = static_cast<Problem*>(h);
  const Space& V = p->mg->space();
  const int ns = (V.k + 1) * (V.k + 2) / 2;
  Vec c(compound_full, compound_full + V.n_compound()), i(interior, interior + V.n_interior());
  std::vector<Real> g(grad, grad + std::size_t(V.mesh->ne()) * 4 * ns);
  std::vector<Real> out = postprocess_velocity(*V.mesh, V, p->opt.nu, c, i, g);
  std::memcpy(post, out.data(), sizeof(double) * out.size());
}

/// measure_errors (inc/postprocess.hpp:142-188) against exact flow kind
/// (1 manufactured, 2 linear): out = (e_u, e_L, e_ustar, div_u).
void orc_mg_errors(void* h, const double* compound_full, const double* interior, const double* grad,
                   const double* post, int kind, double* out) {
  auto* p = static_cast<Problem*>(h);
  const Space& V = p->mg->space();
  const int ns = (V.k + 1) * (V.k + 2) / 2, nh = (V.k + 2) * (V.k + 3) / 2;
  const std::size_t ne = V.mesh->ne();
  Vec c(compound_full, compound_full + V.n_compound()), i(interior, interior + V.n_interior());
  std::vector<Real> g(grad, grad + ne * 4 * ns), ps(post, post + ne * 2 * nh);
  ErrorNorms e = measure_errors(*V.mesh, V, p->opt.nu, c, i, g, ps, kind);
  out[0] = e.e_u;
  out[1] = e.e_L;
  out[2] = e.e_ustar;
  out[3] = e.div_u;
}

/// Element centroids of the finest mesh, [ne][2].
void orc_mg_centroids(void* h, double* out) {
  const Mesh& m = *static_cast<Problem*>(h)->mg->space().mesh;
  for (int e = 0; e < m.ne(); ++e) {
    V2 c(0, 0);
    for (int i = 0; i < 3; ++i) c = c + m.vtx[m.el[e].v[i]];
    out[2 * e] = c.x / 3.0;
    out[2 * e + 1] = c.y / 3.0;
  }
}

/// Manufactured-flow pointwise values for the source-term check
/// (tests/test_postprocess.cpp:44-118): out = u(2), grad u(4), lap u(2),
/// p, grad p(2), stokes_load(nu, beta)(2), ns_load(nu)(2).
void orc_mms_point(double x, double y, double nu, double beta, double* out) {
  const V2 X(x, y);
  const V2 u = mms::velocity(X), l = mms::laplacian(X), gp = mms::pressure_gradient(X);
  Real g[2][2];
  mms::gradient(X, g);
  const V2 fs = mms::stokes_load(nu, beta, X), fn = mms::ns_load(nu, X);
  const double v[15] = {u.x, u.y, g[0][0], g[0][1], g[1][0], g[1][1], l.x, l.y, mms::pressure(X), gp.x, gp.y,
                        fs.x, fs.y, fn.x, fn.y};
  std::memcpy(out, v, sizeof(v));
}

/// navier_stokes_solve (inc/ns.hpp:69-149) for the problem description `p`
/// (mesh, k, nu, inv_eps, bc, load, MG options; wind/beta/mass ignored as in
/// the reference driver). Outputs the final compound velocity, interior
/// coefficients and element pressures. Returns 0, or -1 on a setup error.
int orc_ns_solve(const orc_problem* p, const orc_ns_opts* o, double* velocity, double* interior, double* pressure,
                 orc_ns_report* rep) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    Hierarchy hier = Hierarchy::build(base_mesh(p), p->levels);
    Vec loadcopy;
    Field load;
    if (p->load_kind == 1) {
      int nf = p->base_n << (p->levels - 1);
      loadcopy.assign(p->load, p->load + std::size_t(4) * nf * nf);
      const double* F = loadcopy.data();
      load = [F, nf](const V2& x) { return structured_load(F, nf, x); };
    } else {
      load = make_named_load(p->load_kind, p->nu, p->beta);
    }
    NSOpt no;
    no.picard_tol = o->picard_tol;
    no.newton_rel_tol = o->newton_rel_tol;
    no.newton_abs_tol = o->newton_abs_tol;
    no.max_picard = o->max_picard;
    no.max_newton = o->max_newton;
    no.pseudo_time_inv = o->pseudo_time_inv;
    no.mg.cycle = p->cycle;
    no.mg.smoother = p->smoother;
    no.mg.smooth_steps = p->smooth_steps;
    no.mg.jacobi_damping = p->jacobi_damping;
    no.uzawa.outer_iterations = o->outer_iterations;
    no.uzawa.krylov = {o->rel_tol, o->abs_tol, o->max_iterations};
    NSSolution s = navier_stokes_solve(hier, p->k, make_bc(p->bc_kind), p->nu, load, p->inv_eps, no);
    std::memset(rep, 0, sizeof(*rep));
    rep->picard_iterations = s.report.picard_iterations;
    rep->newton_iterations = s.report.newton_iterations;
    rep->n_picard_inner = int(std::min<std::size_t>(s.report.picard_inner.size(), 512));
    rep->n_newton_inner = int(std::min<std::size_t>(s.report.newton_inner.size(), 256));
    for (int i = 0; i < rep->n_picard_inner; ++i) rep->picard_inner[i] = s.report.picard_inner[i];
    for (int i = 0; i < rep->n_newton_inner; ++i) rep->newton_inner[i] = s.report.newton_inner[i];
    for (std::size_t i = 0; i < s.report.picard_diffs.size() && i < 128; ++i) rep->picard_diffs[i] = s.report.picard_diffs[i];
    for (std::size_t i = 0; i < s.report.newton_diffs.size() && i < 64; ++i) rep->newton_diffs[i] = s.report.newton_diffs[i];
    rep->converged = s.report.converged;
    rep->not_applicable = s.report.not_applicable;
    rep->final_divergence = s.report.final_divergence;
    if (!s.velocity.compound.empty()) {
      std::memcpy(velocity, s.velocity.compound.data(), sizeof(double) * s.velocity.compound.size());
      std::memcpy(interior, s.velocity.interior.data(), sizeof(double) * s.velocity.interior.size());
      std::memcpy(pressure, s.pressure.data(), sizeof(double) * s.pressure.size());
    }
    rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

/// Time `reps` preconditioner applications on a fixed seeded vector (CPU baseline).
double orc_mg_time_apply(void* h, int reps) {
  auto* p = static_cast<Problem*>(h);
  Index n = p->mg->constraints().n_free;
  Vec b(n);
  std::mt19937 rng(47);
  std::uniform_real_distribution<double> d(-1, 1);
  for (auto& v : b) v = d(rng);
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    Vec x = p->mg->apply(b);
    b[0] += 1e-300 * x[0];
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"

extern "C" {
/// The reference tests' random_vec: std::mt19937(seed), uniform(-1, 1)
/// (e.g. reference tests/test_multigrid.cpp:11-17).
void orc_random_vec(long long n, unsigned seed, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (long long i = 0; i < n; ++i) out[i] = dist(rng);
}
}
