// TEST INFRASTRUCTURE: see multigrid.hpp in this directory.
#pragma once
#include "multigrid.hpp"
namespace hdivmg {
struct UzawaOptions {
  int outer_iterations = 2;
  KrylovOptions krylov;
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
}  // namespace hdivmg
