// TEST INFRASTRUCTURE: a reference user's program, written against the
// reference API (hdivmg::MeshHierarchy, AssemblyOptions, MGOptions, pcg,
// uzawa_solve), run twice in one process: once with the reference's own
// hdivmg::MGPreconditioner (the unmodified reference headers over the
// Eigen-API shim) and once with the drop-in hpmg::MGPreconditioner of
// include/hpmg/hdivmg_gpu.hpp (device path through the C ABI). Prints one
// line per comparison and exits non-zero on a mismatch. Built by
// oracle/Makefile (target adapter) where the reference tree exists; run by
// tests/test_gpu_adapter.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <random>

#include "hpmg/hdivmg_gpu.hpp"

using namespace hdivmg;

static double rel(const Vec& a, const Vec& b) { return (a - b).norm() / b.norm(); }

static int fails = 0;
static void check(const char* what, bool ok, double v) {
  std::printf("%-44s %s %.3e\n", what, ok ? "ok  " : "FAIL", v);
  if (!ok) ++fails;
}

template <class Pre>
static LinearOperator matrix_op(const Pre& B) {
  return [&B](const Vec& v) { return Vec(B.matrix() * v); };
}

int main() {
  for (int k : {1, 2, 3}) {
    std::printf("-- k = %d\n", k);
    MeshHierarchy hier = MeshHierarchy::build(unit_square_mesh(4), 3);
    AssemblyOptions opt;
    opt.nu = 1.0;
    opt.beta = 1.0;
    opt.load = [](const Vec2& x) { return Vec2(std::sin(2 * x.x()) + x.y(), std::cos(x.y()) - x.x() * x.x()); };
    VelocityBC bc;
    bc.g = [](const Vec2& x) { return x.y() > 1.0 - 1e-12 ? Vec2(4 * x.x() * (1 - x.x()), 0.0) : Vec2(0, 0); };
    MGOptions mg;
    mg.cycle = CycleKind::V;
    hdivmg::MGPreconditioner R(hier, k, bc, opt, 1e3, mg);
    hpmg::MGPreconditioner G(hier, k, bc, opt, 1e3, mg);
    // interface: sizes, constraints, operator, rhs
    check("constraints().n_free", G.constraints().n_free == R.constraints().n_free, double(G.constraints().n_free));
    check("space().n_compound()", G.space().n_compound() == R.space().n_compound(), double(G.space().n_compound()));
    const SpMat A = G.matrix(), AT = G.matrix_transpose();
    Mat D = Mat(A) - Mat(R.matrix());
    double amax = 0, dmax = 0;
    for (Index j = 0; j < D.cols(); ++j)
      for (Index i = 0; i < D.rows(); ++i) {
        dmax = std::max(dmax, std::abs(D(i, j)));
        amax = std::max(amax, std::abs(R.matrix().coeff(i, j)));
      }
    check("matrix() entrywise / max|A|", dmax <= 1e-13 * amax, dmax / amax);
    check("matrix_transpose() (symmetric: == matrix())", (Mat(AT) - Mat(A)).norm() == 0.0, 0.0);
    check("rhs()", rel(G.rhs(), R.rhs()) < 1e-14, rel(G.rhs(), R.rhs()));
    // one preconditioner application
    Vec b(R.constraints().n_free);
    std::mt19937 rng(3);
    std::uniform_real_distribution<double> u(-1, 1);
    for (Index i = 0; i < b.size(); ++i) b[i] = u(rng);
    check("apply()", rel(G.apply(b), R.apply(b)) < 2e-12, rel(G.apply(b), R.apply(b)));
    // the reference call site pcg(A, M, b, x) unchanged, M on the device
    Vec xr = Vec::Zero(b.size()), xg = Vec::Zero(b.size()), xd = Vec::Zero(b.size());
    SolveStats sr = hdivmg::pcg(matrix_op(R), R.as_operator(), R.rhs(), xr);
    SolveStats sg = hpmg::pcg(hpmg::matrix_operator(G), G.as_operator(), G.rhs(), xg);
    SolveStats sd = hpmg::pcg(G, G.rhs(), xd);  // device-resident loop
    check("pcg(A, M) count vs reference", std::abs(sg.iterations - sr.iterations) <= 1, sg.iterations - sr.iterations);
    check("pcg(B) device loop count vs reference", std::abs(sd.iterations - sr.iterations) <= 1,
          sd.iterations - sr.iterations);
    check("pcg solutions", rel(xg, xr) < 1e-8 && rel(xd, xr) < 1e-8, std::max(rel(xg, xr), rel(xd, xr)));
    // uzawa_solve
    StokesSolution ur = hdivmg::uzawa_solve(R), ug = hpmg::uzawa_solve(G);
    bool same = ur.report.inner_iterations.size() == ug.report.inner_iterations.size();
    for (std::size_t i = 0; same && i < ur.report.inner_iterations.size(); ++i)
      same = std::abs(ur.report.inner_iterations[i] - ug.report.inner_iterations[i]) <= 1;
    check("uzawa_solve inner counts", same, double(ug.report.inner_iterations[0]));
    check("uzawa_solve velocity", rel(ug.velocity, ur.velocity) < 1e-9, rel(ug.velocity, ur.velocity));
  }
  std::printf("%s\n", fails ? "adapter: FAILED" : "adapter: all checks passed");
  return fails ? 1 : 0;
}
