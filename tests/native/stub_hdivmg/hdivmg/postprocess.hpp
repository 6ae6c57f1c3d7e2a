// TEST INFRASTRUCTURE: see multigrid.hpp in this directory.
#pragma once
#include "multigrid.hpp"
namespace hdivmg {
struct PostprocessedVelocity {
  int k_hi = 1;
  Mat coeffs;
};
struct ErrorNorms {
  Real e_u = 0, e_L = 0, e_ustar = 0, div_u = 0;
};
}  // namespace hdivmg
