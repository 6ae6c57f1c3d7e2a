// TEST INFRASTRUCTURE: a declaration-only stand-in for the reference headers
// (Eigen is absent from this image), shaped after proj/include/hdivmg/*.hpp,
// so that include/hpmg/hdivmg_gpu.hpp can be compiled (-fsyntax-only) here.
// Only the members the adapter touches are declared.
#pragma once
#include <functional>
#include <vector>

namespace hdivmg {
using Real = double;
using Index = long;
struct Vec {
  std::vector<double> v;
  Vec() = default;
  explicit Vec(Index n) : v(size_t(n)) {}
  static Vec Zero(Index n) { return Vec(n); }
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  Index size() const { return Index(v.size()); }
  void resize(Index n) { v.resize(size_t(n)); }
};
struct Vec2 {
  double a = 0, b = 0;
  Vec2(double x, double y) : a(x), b(y) {}
  double x() const { return a; }
  double y() const { return b; }
};
struct Mat {
  Mat() = default;
  Mat(Index r, Index c) : rows(r), d(size_t(r * c)) {}
  double& operator()(Index i, Index j) { return d[size_t(j * rows + i)]; }
  double* data() { return d.data(); }
  const double* data() const { return d.data(); }
  static Mat Zero(Index r, Index c) { return Mat(r, c); }
  Index rows = 0;
  std::vector<double> d;
};
struct Mat2 {
  double m[4] = {0, 0, 0, 0};
  double operator()(int i, int j) const { return m[2 * i + j]; }
};
struct Triplet {
  Triplet(int r, int c, double v) : r(r), c(c), v(v) {}
  int r, c;
  double v;
};
struct SpMat {
  SpMat(int, int) {}
  template <class It>
  void setFromTriplets(It, It) {}
};
using LinearOperator = std::function<Vec(const Vec&)>;
namespace bc {
constexpr int kOutflow = 2;
}
struct Facet {
  int a, b, tag;
};
struct Element {
  int v[3];
};
struct Mesh {
  std::vector<Vec2> vertices;
  std::vector<Element> elements;
  std::vector<Facet> facets;
  int nv() const { return int(vertices.size()); }
  int ne() const { return int(elements.size()); }
};
struct MeshHierarchy {
  std::vector<Mesh> levels;
};
struct CompoundSpace {
  CompoundSpace() = default;
  CompoundSpace(const Mesh&, int order) : k(order) {}
  Index n_compound() const { return 0; }
  int k = 0;
};
struct HDGVelocity {
  CompoundSpace V;
  Vec compound, interior;
};
struct VelocityBC {
  std::function<Vec2(const Vec2&)> g;
};
struct AssemblyOptions {
  Real nu = 1, beta = 0, mass_coef = 0;
  std::function<Vec2(const Vec2&)> load;
  const HDGVelocity* advection = nullptr;
  bool newton = false;
  const HDGVelocity* mass_field = nullptr;
};
enum class CycleKind { V, W, VariableV };
enum class SmootherKind { Multiplicative, Additive };
struct MGOptions {
  CycleKind cycle = CycleKind::W;
  SmootherKind smoother = SmootherKind::Multiplicative;
  int smooth_steps = 1;
  Real jacobi_damping = 1.0 / 3.0;
};
struct KrylovOptions {
  Real rel_tol = 1e-8, abs_tol = 1e-10;
  int max_iterations = 500;
};
struct SolveStats {
  int iterations = 0;
  bool converged = false, not_applicable = false;
  Real residual = 0;
};
struct LocalSolution {
  Vec interior, p_ortho;
  Mat grad_coeffs;
};
}  // namespace hdivmg
