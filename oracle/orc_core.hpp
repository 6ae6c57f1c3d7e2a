// TEST INFRASTRUCTURE ONLY. CPU restatement ("oracle") of the hdivmg reference
// library, used solely by tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs as the checker. The product path
// (paper_2303_06762_b200/) never links or calls anything under oracle/.
//
// Parity status: the reference cannot be compiled here (Eigen 3, Catch2 and
// CLI11 are absent), so this restatement is pinned by the reference's own
// known-answer tests (CR congruence, dense Schur complement, transfer and
// smoother identities, paper iteration-count tables), see tests/test_oracle_*.
//
// This file: dense linear algebra (partial/full pivot LU, one-sided Jacobi
// SVD), polynomials and quadrature. Eigen-free; row-major dense storage.
#pragma once

#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <cstdint>
#include <functional>
#include <numeric>
#include <stdexcept>
#include <vector>

namespace orc {

#ifdef ORC_REAL
using Real = ORC_REAL;  // extended-precision diagnostic build (oracle/hp_solve.cpp)
#else
using Real = double;
#endif
using Index = std::int64_t;
using Vec = std::vector<Real>;

struct V2 {
  Real x = 0, y = 0;
  V2() = default;
  V2(Real a, Real b) : x(a), y(b) {}
  V2 operator+(const V2& o) const { return {x + o.x, y + o.y}; }
  V2 operator-(const V2& o) const { return {x - o.x, y - o.y}; }
  V2 operator*(Real s) const { return {x * s, y * s}; }
  V2 operator/(Real s) const { return {x / s, y / s}; }
  V2& operator+=(const V2& o) { x += o.x; y += o.y; return *this; }
  V2& operator-=(const V2& o) { x -= o.x; y -= o.y; return *this; }
  Real dot(const V2& o) const { return x * o.x + y * o.y; }
  Real norm() const { return std::sqrt(x * x + y * y); }
  V2 normalized() const { Real n = norm(); return {x / n, y / n}; }
};
inline V2 operator*(Real s, const V2& v) { return {s * v.x, s * v.y}; }

using Field = std::function<V2(const V2&)>;

// ---------------------------------------------------------------- dense ----
struct Mat {
  int r = 0, c = 0;
  std::vector<Real> a;
  Mat() = default;
  Mat(int rows, int cols) : r(rows), c(cols), a(std::size_t(rows) * cols, 0.0) {}
  Real& operator()(int i, int j) { return a[std::size_t(i) * c + j]; }
  Real operator()(int i, int j) const { return a[std::size_t(i) * c + j]; }
  static Mat eye(int n) { Mat m(n, n); for (int i = 0; i < n; ++i) m(i, i) = 1; return m; }
  Mat t() const { Mat m(c, r); for (int i = 0; i < r; ++i) for (int j = 0; j < c; ++j) m(j, i) = (*this)(i, j); return m; }
};

inline Mat matmul(const Mat& A, const Mat& B) {
  assert(A.c == B.r);
  Mat C(A.r, B.c);
  for (int i = 0; i < A.r; ++i)
    for (int k = 0; k < A.c; ++k) {
      Real s = A(i, k);
      if (s == 0.0) continue;
      for (int j = 0; j < B.c; ++j) C(i, j) += s * B(k, j);
    }
  return C;
}

inline Vec matvec(const Mat& A, const Vec& x) {
  Vec y(A.r, 0.0);
  for (int i = 0; i < A.r; ++i) {
    Real s = 0;
    for (int j = 0; j < A.c; ++j) s += A(i, j) * x[j];
    y[i] = s;
  }
  return y;
}

inline Real dot(const Vec& a, const Vec& b) {
  Real s = 0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
inline Real norm(const Vec& a) { return std::sqrt(dot(a, a)); }

/// LU with partial (row) pivoting, P A = L U. Follows the role of
/// Eigen::PartialPivLU at reference inc/smoother.hpp:99, inc/assembly.hpp:359,
/// inc/multigrid.hpp:87, inc/transfer.hpp:124.
struct LU {
  int n = 0;
  Mat f;                 // packed L (unit diag) and U
  std::vector<int> piv;  // row permutation: row i of PA = row piv[i] of A
  LU() = default;
  explicit LU(const Mat& A) { factor(A); }
  /// Diagnostic variant (ORC_VARIANT, orc_mg.hpp): solves by an explicit
  /// inverse (columns solve(e_j)) applied as a mat-vec, the device's
  /// formulation, to measure how much that arithmetic alone moves results.
  Mat inv;
  bool use_inv = false;
  void make_inverse() {
    Mat X(n, n);
    for (int j = 0; j < n; ++j) {
      Vec e(n, 0.0);
      e[j] = 1.0;
      Vec c = solve(e);
      for (int i = 0; i < n; ++i) X(i, j) = c[i];
    }
    inv = X;
    use_inv = true;
  }
  void factor(const Mat& A) {
    assert(A.r == A.c);
    n = A.r;
    f = A;
    piv.resize(n);
    std::iota(piv.begin(), piv.end(), 0);
    for (int k = 0; k < n; ++k) {
      int p = k;
      Real best = std::abs(f(k, k));
      for (int i = k + 1; i < n; ++i)
        if (std::abs(f(i, k)) > best) { best = std::abs(f(i, k)); p = i; }
      if (p != k) {
        for (int j = 0; j < n; ++j) std::swap(f(k, j), f(p, j));
        std::swap(piv[k], piv[p]);
      }
      Real d = f(k, k);
      if (d == 0.0) continue;
      for (int i = k + 1; i < n; ++i) {
        Real l = f(i, k) / d;
        f(i, k) = l;
        if (l == 0.0) continue;
        for (int j = k + 1; j < n; ++j) f(i, j) -= l * f(k, j);
      }
    }
  }
  Vec solve(const Vec& b) const {
    if (use_inv) {
      Vec x(n, 0.0);
      for (int i = 0; i < n; ++i) {
        Real s = 0;
        for (int j = 0; j < n; ++j) s += inv(i, j) * b[j];
        x[i] = s;
      }
      return x;
    }
    Vec y(n);
    for (int i = 0; i < n; ++i) y[i] = b[piv[i]];
    for (int i = 0; i < n; ++i) {
      Real s = y[i];
      for (int j = 0; j < i; ++j) s -= f(i, j) * y[j];
      y[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
      Real s = y[i];
      for (int j = i + 1; j < n; ++j) s -= f(i, j) * y[j];
      y[i] = s / f(i, i);
    }
    return y;
  }
  /// Solves A^T x = b (reference inc/smoother.hpp:88, lu.transpose().solve).
  Vec solve_t(const Vec& b) const {
    if (use_inv) {
      Vec x(n, 0.0);
      for (int i = 0; i < n; ++i) {
        Real s = 0;
        for (int j = 0; j < n; ++j) s += inv(j, i) * b[j];
        x[i] = s;
      }
      return x;
    }
    // A^T = U^T L^T P  =>  U^T z = b, L^T w = z, x = P^T w
    Vec z(b);
    for (int i = 0; i < n; ++i) {
      Real s = z[i];
      for (int j = 0; j < i; ++j) s -= f(j, i) * z[j];
      z[i] = s / f(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      Real s = z[i];
      for (int j = i + 1; j < n; ++j) s -= f(j, i) * z[j];
      z[i] = s;
    }
    Vec x(n);
    for (int i = 0; i < n; ++i) x[piv[i]] = z[i];
    return x;
  }
  Mat solve(const Mat& B) const {
    Mat X(B.r, B.c);
    Vec col(B.r);
    for (int j = 0; j < B.c; ++j) {
      for (int i = 0; i < B.r; ++i) col[i] = B(i, j);
      Vec s = solve(col);
      for (int i = 0; i < B.r; ++i) X(i, j) = s[i];
    }
    return X;
  }
};

/// LU with complete pivoting; square systems only (role of Eigen::FullPivLU
/// at reference inc/fespace.hpp:181).
struct FullLU {
  int n = 0;
  Mat f;
  std::vector<int> prow, pcol;
  int rank = 0;
  explicit FullLU(const Mat& A) {
    n = A.r;
    f = A;
    prow.resize(n);
    pcol.resize(n);
    std::iota(prow.begin(), prow.end(), 0);
    std::iota(pcol.begin(), pcol.end(), 0);
    Real maxpivot = 0;
    for (int k = 0; k < n; ++k) {
      int pi = k, pj = k;
      Real best = -1;
      for (int i = k; i < n; ++i)
        for (int j = k; j < n; ++j)
          if (std::abs(f(i, j)) > best) { best = std::abs(f(i, j)); pi = i; pj = j; }
      if (k == 0) maxpivot = best;
      if (best <= 1e-14 * maxpivot || best == 0.0) break;
      rank = k + 1;
      if (pi != k) { for (int j = 0; j < n; ++j) std::swap(f(k, j), f(pi, j)); std::swap(prow[k], prow[pi]); }
      if (pj != k) { for (int i = 0; i < n; ++i) std::swap(f(i, k), f(i, pj)); std::swap(pcol[k], pcol[pj]); }
      for (int i = k + 1; i < n; ++i) {
        Real l = f(i, k) / f(k, k);
        f(i, k) = l;
        for (int j = k + 1; j < n; ++j) f(i, j) -= l * f(k, j);
      }
    }
  }
  bool invertible() const { return rank == n; }
  Vec solve(const Vec& b) const {
    Vec y(n);
    for (int i = 0; i < n; ++i) y[i] = b[prow[i]];
    for (int i = 0; i < n; ++i) for (int j = 0; j < i; ++j) y[i] -= f(i, j) * y[j];
    for (int i = n - 1; i >= 0; --i) {
      for (int j = i + 1; j < n; ++j) y[i] -= f(i, j) * y[j];
      y[i] /= f(i, i);
    }
    Vec x(n);
    for (int i = 0; i < n; ++i) x[pcol[i]] = y[i];
    return x;
  }
};

/// Singular value decomposition A = U S V^T by one-sided Jacobi (Hestenes)
/// rotations on the columns of A; V is the full n x n orthogonal factor and
/// the singular values are sorted descending (role of Eigen::JacobiSVD with
/// ComputeFullV at reference inc/fespace.hpp:152,155).
struct SVD {
  int m = 0, n = 0;
  Mat V;          // n x n, columns sorted by descending singular value
  Vec s;          // n singular values (descending; trailing zeros)
  Mat B;          // m x n, A V (columns = s_j u_j)
  explicit SVD(const Mat& A) {
    m = A.r;
    n = A.c;
    B = A;
    V = Mat::eye(n);
    for (int sweep = 0; sweep < 60; ++sweep) {
      Real off = 0;
      for (int p = 0; p < n - 1; ++p)
        for (int q = p + 1; q < n; ++q) {
          Real alpha = 0, beta = 0, gamma = 0;
          for (int i = 0; i < m; ++i) {
            alpha += B(i, p) * B(i, p);
            beta += B(i, q) * B(i, q);
            gamma += B(i, p) * B(i, q);
          }
          if (gamma == 0.0) continue;
          Real rel = std::abs(gamma) / std::sqrt(std::max(alpha * beta, Real(1e-300)));
          off = std::max(off, rel);
          if (rel < 1e-16) continue;
          Real zeta = (beta - alpha) / (2 * gamma);
          Real t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1 + zeta * zeta));
          Real cs = 1 / std::sqrt(1 + t * t), sn = cs * t;
          for (int i = 0; i < m; ++i) {
            Real bp = B(i, p), bq = B(i, q);
            B(i, p) = cs * bp - sn * bq;
            B(i, q) = sn * bp + cs * bq;
          }
          for (int i = 0; i < n; ++i) {
            Real vp = V(i, p), vq = V(i, q);
            V(i, p) = cs * vp - sn * vq;
            V(i, q) = sn * vp + cs * vq;
          }
        }
      if (off < 1e-15) break;
    }
    s.assign(n, 0);
    for (int j = 0; j < n; ++j) {
      Real acc = 0;
      for (int i = 0; i < m; ++i) acc += B(i, j) * B(i, j);
      s[j] = std::sqrt(acc);
    }
    std::vector<int> ord(n);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return s[a] > s[b]; });
    Mat V2(n, n), B2(m, n);
    Vec s2(n);
    for (int j = 0; j < n; ++j) {
      s2[j] = s[ord[j]];
      for (int i = 0; i < n; ++i) V2(i, j) = V(i, ord[j]);
      for (int i = 0; i < m; ++i) B2(i, j) = B(i, ord[j]);
    }
    V = V2;
    B = B2;
    s = s2;
  }
  /// Minimum-norm least-squares solution (role of JacobiSVD::solve).
  Vec solve(const Vec& b) const {
    Vec x(n, 0.0);
    Real thr = (s.empty() ? 0 : s[0]) * 1e-13;
    for (int j = 0; j < n; ++j) {
      if (s[j] <= thr || s[j] == 0.0) continue;
      Real c = 0;
      for (int i = 0; i < m; ++i) c += B(i, j) * b[i];
      c /= s[j] * s[j];
      for (int i = 0; i < n; ++i) x[i] += c * V(i, j);
    }
    return x;
  }
};

// ---------------------------------------------------------- polynomials ----
/// Legendre L_0..L_k at t (reference inc/polynomial.hpp:12-17).
inline void legendre_all(int k, Real t, Real* out) {
  out[0] = 1.0;
  if (k >= 1) out[1] = t;
  for (int j = 2; j <= k; ++j) out[j] = ((2 * j - 1) * t * out[j - 1] - (j - 1) * out[j - 2]) / j;
}
inline Real legendre(int i, Real t) {
  Real v[16];
  legendre_all(i, t, v);
  return v[i];
}

/// Bivariate polynomial in monomial coefficients; x^i y^j at (i+j)(i+j+1)/2+j
/// (reference inc/polynomial.hpp:27-131).
struct Poly {
  int deg = 0;
  std::vector<Real> c{0.0};
  Poly() = default;
  explicit Poly(int d) : deg(d), c(std::size_t(dim(d)), 0.0) {}
  static int dim(int d) { return (d + 1) * (d + 2) / 2; }
  static int idx(int i, int j) { int s = i + j; return s * (s + 1) / 2 + j; }
  static Poly mono(int i, int j) { Poly p(i + j); p.c[idx(i, j)] = 1.0; return p; }
  Real coef(int i, int j) const { return (i + j <= deg) ? c[idx(i, j)] : 0.0; }
  Real eval(Real x, Real y) const {
    Real sum = 0;
    for (int s = 0; s <= deg; ++s)
      for (int j = 0; j <= s; ++j) {
        Real v = c[idx(s - j, j)];
        if (v != 0.0) sum += v * std::pow(x, s - j) * std::pow(y, j);
      }
    return sum;
  }
  Poly dx() const {
    Poly p(std::max(0, deg - 1));
    for (int s = 1; s <= deg; ++s)
      for (int j = 0; j <= s; ++j) {
        int i = s - j;
        if (i >= 1) p.c[idx(i - 1, j)] += i * c[idx(i, j)];
      }
    return p;
  }
  Poly dy() const {
    Poly p(std::max(0, deg - 1));
    for (int s = 1; s <= deg; ++s)
      for (int j = 1; j <= s; ++j) p.c[idx(s - j, j - 1)] += j * c[idx(s - j, j)];
    return p;
  }
  void grow(int d) {
    if (d <= deg) return;
    c.resize(std::size_t(dim(d)), 0.0);
    deg = d;
  }
  Poly& operator+=(const Poly& o) {
    grow(o.deg);
    for (std::size_t i = 0; i < o.c.size(); ++i) c[i] += o.c[i];
    return *this;
  }
  Poly& operator-=(const Poly& o) {
    grow(o.deg);
    for (std::size_t i = 0; i < o.c.size(); ++i) c[i] -= o.c[i];
    return *this;
  }
  Poly& operator*=(Real a) { for (auto& v : c) v *= a; return *this; }
};
inline Poly operator+(Poly a, const Poly& b) { return a += b; }
inline Poly operator-(Poly a, const Poly& b) { return a -= b; }
inline Poly operator*(Real s, Poly p) { return p *= s; }
inline Poly operator*(const Poly& a, const Poly& b) {
  Poly p(a.deg + b.deg);
  for (int sa = 0; sa <= a.deg; ++sa)
    for (int ja = 0; ja <= sa; ++ja) {
      Real ca = a.c[Poly::idx(sa - ja, ja)];
      if (ca == 0.0) continue;
      for (int sb = 0; sb <= b.deg; ++sb)
        for (int jb = 0; jb <= sb; ++jb) {
          Real cb = b.c[Poly::idx(sb - jb, jb)];
          if (cb != 0.0) p.c[Poly::idx(sa - ja + sb - jb, ja + jb)] += ca * cb;
        }
    }
  return p;
}

/// a! b! / (a+b+2)! in extended precision (reference inc/polynomial.hpp:158-163).
inline long double tri_mono_ld(int a, int b) {
  long double binom = 1.0L;
  for (int i = 1; i <= a; ++i) binom *= static_cast<long double>(b + i) / i;
  return 1.0L / (binom * (a + b + 1) * (a + b + 2));
}

/// Reference-triangle L2 product accumulated in long double
/// (reference inc/polynomial.hpp:178-195).
inline Real tri_l2(const Poly& a, const Poly& b) {
  long double sum = 0.0L;
  for (int sa = 0; sa <= a.deg; ++sa)
    for (int ja = 0; ja <= sa; ++ja) {
      Real ca = a.c[Poly::idx(sa - ja, ja)];
      if (ca == 0.0) continue;
      for (int sb = 0; sb <= b.deg; ++sb)
        for (int jb = 0; jb <= sb; ++jb) {
          Real cb = b.c[Poly::idx(sb - jb, jb)];
          if (cb == 0.0) continue;
          sum += static_cast<long double>(ca) * cb * tri_mono_ld(sa + sb - ja - jb, ja + jb);
        }
    }
  return static_cast<Real>(sum);
}

/// Orthonormal P^k on the reference triangle, four Gram-Schmidt passes
/// (reference inc/polynomial.hpp:239-256 ... :199-214 in the file's own numbering).
inline std::vector<Poly> orthonormal_basis(int k) {
  std::vector<Poly> basis;
  for (int s = 0; s <= k; ++s)
    for (int j = 0; j <= s; ++j) {
      Poly v = Poly::mono(s - j, j);
      for (int pass = 0; pass < 4; ++pass) {
        for (const Poly& q : basis) v -= tri_l2(v, q) * q;
        Real nrm = std::sqrt(tri_l2(v, v));
        v *= 1.0 / nrm;
      }
      basis.push_back(v);
    }
  return basis;
}

// ----------------------------------------------------------- quadrature ----
struct LineRule {
  Vec pts, wts;
};

/// Gauss-Legendre on [-1,1] by Newton from a Chebyshev guess
/// (reference inc/quadrature.hpp:18-50).
inline LineRule line_rule(int degree) {
  const int n = std::max(1, (degree + 2) / 2);
  LineRule r;
  r.pts.resize(n);
  r.wts.resize(n);
  auto eval = [n](Real x, Real& p1, Real& p0) {
    p0 = 1.0;
    p1 = x;
    for (int j = 2; j <= n; ++j) {
      Real p2 = ((2 * j - 1) * x * p1 - (j - 1) * p0) / j;
      p0 = p1;
      p1 = p2;
    }
  };
  for (int i = 0; i < n; ++i) {
    Real x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      Real p1, p0;
      eval(x, p1, p0);
      Real dp = n * (x * p1 - p0) / (x * x - 1.0);
      Real dx = p1 / dp;
      x -= dx;
      if (std::abs(dx) < 1e-16) break;
    }
    Real p1, p0;
    eval(x, p1, p0);
    Real dp = n * (x * p1 - p0) / (x * x - 1.0);
    r.pts[n - 1 - i] = x;
    r.wts[n - 1 - i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
  return r;
}

struct TriRule {
  std::vector<V2> pts;
  Vec wts;
};

/// Collapsed (Duffy) tensor Gauss rule on (0,0)-(1,0)-(0,1)
/// (reference inc/quadrature.hpp:61-79).
inline TriRule tri_rule(int degree) {
  LineRule gu = line_rule(degree + 1), gv = line_rule(degree);
  TriRule r;
  for (std::size_t i = 0; i < gu.pts.size(); ++i) {
    Real u = 0.5 * (gu.pts[i] + 1.0), wu = 0.5 * gu.wts[i];
    for (std::size_t j = 0; j < gv.pts.size(); ++j) {
      Real v = 0.5 * (gv.pts[j] + 1.0), wv = 0.5 * gv.wts[j];
      r.pts.emplace_back(u * (1.0 - v), u * v);
      r.wts.push_back(wu * wv * u);
    }
  }
  return r;
}

}  // namespace orc
