// TEST INFRASTRUCTURE ONLY (diagnostic). The restatement compiled with
// Real = long double (64-bit mantissa): assembles one seeded unit-square
// Stokes problem and runs uzawa_solve, writing the final full velocity (as
// double) to a file. Used to decide which of two double-precision solutions
// (device, reference) is closer to the exact discrete solution when they
// differ by more than round-off (tools/hp_floor.py).
//   usage: hp_solve base_n levels k beta inv_eps seed out.bin
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
  const int n = base_n << (levels - 1);
  std::vector<double> F(std::size_t(4) * n * n);
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (auto& v : F) v = dist(rng);
  Hierarchy hier = Hierarchy::build(unit_square(base_n), levels);
  AsmOpt opt;
  opt.nu = 1.0;
  opt.beta = beta;
  opt.load = [&](const V2& x) {
    const double xx = double(x.x), yy = double(x.y);
    int i = std::min(n - 1, std::max(0, int(std::floor(xx * n))));
    int j = std::min(n - 1, std::max(0, int(std::floor(yy * n))));
    bool lower = (xx - double(i) / n) >= (yy - double(j) / n);
    std::size_t s = (std::size_t(j) * n + i) * 2 + (lower ? 0 : 1);
    return V2(F[2 * s], F[2 * s + 1]);
  };
  MGOpt mo;
  mo.cycle = kV;
  MG mg(hier, k, nullptr, opt, inv_eps, mo);
  UzawaOpt uo;
  StokesSolution s = uzawa(mg, uo);
  std::vector<double> v(s.velocity.begin(), s.velocity.end());
  FILE* f = std::fopen(argv[7], "wb");
  std::fwrite(v.data(), sizeof(double), v.size(), f);
  std::fclose(f);
  std::printf("%d %d\n", s.report.inner_iterations.size() > 0 ? s.report.inner_iterations[0] : -1,
              s.report.inner_iterations.size() > 1 ? s.report.inner_iterations[1] : -1);
  return 0;
}
