// TEST INFRASTRUCTURE ONLY (diagnostic). The restatement compiled with
// Real = long double (64-bit mantissa): assembles one seeded unit-square
// Stokes problem and runs uzawa_solve, writing the final full velocity (as
// double) to a file. Used to decide which of two double-precision solutions
// (device, reference) is closer to the exact discrete solution when they
// differ by more than round-off (tools/hp_floor.py).
//   usage: hp_solve base_n levels k beta inv_eps seed out.bin
//          [nu lo hi wind bc restart]   (wind 2: config-5 curl field, bc 4:
//          lid (1,0) on y = 1; restart: GMRES(m), 0 unrestarted)
#include <cstdio>
#include <cstdlib>
#include <random>

#include "orc_mg.hpp"

using namespace orc;

int main(int argc, char** argv) {
  if (argc < 8) return 2;
  const int base_n = std::atoi(argv[1]), levels = std::atoi(argv[2]), k = std::atoi(argv[3]);
  const double beta = std::atof(argv[4]), inv_eps = std::atof(argv[5]);
  const unsigned seed = unsigned(std::atoi(argv[6]));
  const double nu = argc > 8 ? std::atof(argv[8]) : 1.0;
  const double lo = argc > 9 ? std::atof(argv[9]) : -1.0, hi = argc > 10 ? std::atof(argv[10]) : 1.0;
  const int wind = argc > 11 ? std::atoi(argv[11]) : 0, bc = argc > 12 ? std::atoi(argv[12]) : 0;
  const int restart = argc > 13 ? std::atoi(argv[13]) : 0;
  const int n = base_n << (levels - 1);
  std::vector<double> F(std::size_t(4) * n * n);
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (auto& v : F) v = dist(rng);
  Hierarchy hier = Hierarchy::build(unit_square(base_n), levels);
  AsmOpt opt;
  opt.nu = nu;
  opt.beta = beta;
  opt.load = [&](const V2& x) {
    const double xx = double(x.x), yy = double(x.y);
    int i = std::min(n - 1, std::max(0, int(std::floor(xx * n))));
    int j = std::min(n - 1, std::max(0, int(std::floor(yy * n))));
    bool lower = (xx - double(i) / n) >= (yy - double(j) / n);
    std::size_t s = (std::size_t(j) * n + i) * 2 + (lower ? 0 : 1);
    return V2(F[2 * s], F[2 * s + 1]);
  };
  HDGVel w;
  if (wind == 2) {  // curl of sin^2(pi x) sin^2(pi y)
    w = interpolate_hdg(hier.levels.back(), k, [](const V2& x) {
      const Real s = std::sin(Real(M_PI) * x.x), t = std::sin(Real(M_PI) * x.y);
      return V2(Real(M_PI) * s * s * std::sin(2 * Real(M_PI) * x.y), -Real(M_PI) * std::sin(2 * Real(M_PI) * x.x) * t * t);
    });
    opt.advection = &w;
  }
  Field g = nullptr;
  if (bc == 4) g = [](const V2& x) { return x.y > 1.0 - 1e-12 ? V2(1.0, 0.0) : V2(0, 0); };
  MGOpt mo;
  mo.cycle = kV;
  MG mg(hier, k, g, opt, inv_eps, mo);
  UzawaOpt uo;
  uo.krylov.restart = restart;
  StokesSolution s = uzawa(mg, uo);
  std::vector<double> v(s.velocity.begin(), s.velocity.end());
  FILE* f = std::fopen(argv[7], "wb");
  std::fwrite(v.data(), sizeof(double), v.size(), f);
  std::fclose(f);
  std::printf("%d %d\n", s.report.inner_iterations.size() > 0 ? s.report.inner_iterations[0] : -1,
              s.report.inner_iterations.size() > 1 ? s.report.inner_iterations[1] : -1);
  return 0;
}
