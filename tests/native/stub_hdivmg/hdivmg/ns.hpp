// TEST INFRASTRUCTURE: see multigrid.hpp in this directory.
#pragma once
#include "uzawa.hpp"
namespace hdivmg {
struct NSOptions {
  Real picard_tol = 1e-4, newton_rel_tol = 1e-8, newton_abs_tol = 1e-10;
  int max_picard = 60, max_newton = 25;
  Real pseudo_time_inv = 0.0;
  MGOptions mg;
  UzawaOptions uzawa;
};
struct NSReport {
  int picard_iterations = 0, newton_iterations = 0;
  std::vector<int> picard_inner, newton_inner;
  std::vector<Real> picard_diffs, newton_diffs;
  bool converged = false, not_applicable = false;
  Real final_divergence = 0;
};
struct NSSolution {
  HDGVelocity velocity;
  Vec pressure;
  LocalSolution locals;
  NSReport report;
};
}  // namespace hdivmg
