// Host-side per-order reference data for the element condensation kernels:
// the hierarchical RT_k basis on the reference triangle and its contractions
// with the orthonormal P^k basis, tabulated once per order k and uploaded.
//
// The basis follows the reference definition (reference inc/fespace.hpp:44-228):
//   facet function (e,0): RT0 scaled so its normal trace on edge e is 1;
//   facet function (e,i>=1): normal trace exactly L_i on edge e, 0 elsewhere,
//     divergence-free, L2-orthogonal to the divergence-free bubbles;
//   interior functions: divergence-free bubbles (G-normalised) then the
//     min-norm preimages of the zero-mean scalar modes under div.
// Null spaces and min-norm solves use Householder QR here (the reference uses
// JacobiSVD); all spans and the min-norm preimages are basis-independent, so
// the condensed operator agrees to round-off (only the bubble basis rotation
// within its span may differ, which the Schur complement does not see).
//
// Because the element map is affine, every volume/edge integral of the
// Stokes-type forms factors into a reference tensor contracted with J, J^-1
// and the facet orientation factors; the kernels only do those contractions.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <vector>

namespace hpmg {
namespace host {

// ------------------------------------------------------------- polynomials
struct Poly {  // coefficients of x^i y^j at (i+j)(i+j+1)/2 + j
  int deg = 0;
  std::vector<double> c = std::vector<double>(1, 0.0);
  static int dim(int d) { return (d + 1) * (d + 2) / 2; }
  static int at(int i, int j) { return (i + j) * (i + j + 1) / 2 + j; }
  static Poly zero(int d) { Poly p; p.deg = d; p.c.assign(dim(d), 0.0); return p; }
  static Poly mono(int i, int j) { Poly p = zero(i + j); p.c[at(i, j)] = 1.0; return p; }
  double get(int i, int j) const { return i + j <= deg ? c[at(i, j)] : 0.0; }
  void widen(int d) { if (d > deg) { c.resize(dim(d), 0.0); deg = d; } }
  void axpy(double a, const Poly& o) { widen(o.deg); for (size_t i = 0; i < o.c.size(); ++i) c[i] += a * o.c[i]; }
  Poly mul(const Poly& o) const {
    Poly p = zero(deg + o.deg);
    for (int s = 0; s <= deg; ++s)
      for (int j = 0; j <= s; ++j) {
        double a = c[at(s - j, j)];
        if (a == 0.0) continue;
        for (int t = 0; t <= o.deg; ++t)
          for (int l = 0; l <= t; ++l) {
            double b = o.c[at(t - l, l)];
            if (b != 0.0) p.c[at(s - j + t - l, j + l)] += a * b;
          }
      }
    return p;
  }
  Poly dx() const {
    Poly p = zero(deg > 0 ? deg - 1 : 0);
    for (int s = 1; s <= deg; ++s)
      for (int j = 0; j < s; ++j) p.c[at(s - j - 1, j)] += (s - j) * c[at(s - j, j)];
    return p;
  }
  Poly dy() const {
    Poly p = zero(deg > 0 ? deg - 1 : 0);
    for (int s = 1; s <= deg; ++s)
      for (int j = 1; j <= s; ++j) p.c[at(s - j, j - 1)] += j * c[at(s - j, j)];
    return p;
  }
  double operator()(double x, double y) const {
    double sum = 0.0;
    for (int s = 0; s <= deg; ++s)
      for (int j = 0; j <= s; ++j) {
        double a = c[at(s - j, j)];
        if (a != 0.0) sum += a * std::pow(x, s - j) * std::pow(y, j);
      }
    return sum;
  }
};

/// exact int_T x^a y^b = a! b! / (a+b+2)!, extended precision
inline long double mono_int(int a, int b) {
  long double r = 1.0L;
  for (int i = 1; i <= a; ++i) r *= (long double)(b + i) / i;
  return 1.0L / (r * (a + b + 1) * (a + b + 2));
}
inline double l2(const Poly& p, const Poly& q) {
  long double s = 0.0L;
  for (int a = 0; a <= p.deg; ++a)
    for (int i = 0; i <= a; ++i) {
      double u = p.c[Poly::at(a - i, i)];
      if (u == 0.0) continue;
      for (int b = 0; b <= q.deg; ++b)
        for (int j = 0; j <= b; ++j) {
          double v = q.c[Poly::at(b - j, j)];
          if (v != 0.0) s += (long double)u * v * mono_int(a - i + b - j, i + j);
        }
    }
  return double(s);
}
/// orthonormal P^k by degree, four Gram-Schmidt passes (reference inc/polynomial.hpp:178-195)
inline std::vector<Poly> onb(int k) {
  std::vector<Poly> B;
  for (int s = 0; s <= k; ++s)
    for (int j = 0; j <= s; ++j) {
      Poly v = Poly::mono(s - j, j);
      for (int pass = 0; pass < 4; ++pass) {
        for (const Poly& q : B) v.axpy(-l2(v, q), q);
        double n = std::sqrt(l2(v, v));
        for (double& t : v.c) t /= n;
      }
      B.push_back(v);
    }
  return B;
}
inline void legendre(int k, double t, double* L) {
  L[0] = 1.0;
  if (k >= 1) L[1] = t;
  for (int j = 2; j <= k; ++j) L[j] = ((2 * j - 1) * t * L[j - 1] - (j - 1) * L[j - 2]) / j;
}

// -------------------------------------------------------------- quadrature
/// Gauss-Legendre on [-1,1], exact to degree 2n-1 with n = max(1,(deg+2)/2)
/// (same rule as reference inc/quadrature.hpp:18-50).
inline void gauss(int degree, std::vector<double>& x, std::vector<double>& w) {
  const int n = std::max(1, (degree + 2) / 2);
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5)), p1 = 0, p0 = 0, dp = 0;
    for (int it = 0; it <= 100; ++it) {
      p0 = 1.0;
      p1 = t;
      for (int j = 2; j <= n; ++j) {
        double p2 = ((2 * j - 1) * t * p1 - (j - 1) * p0) / j;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (t * p1 - p0) / (t * t - 1.0);
      if (it == 100) break;
      double dt = p1 / dp;
      t -= dt;
      if (std::abs(dt) < 1e-16) {
        p0 = 1.0;
        p1 = t;
        for (int j = 2; j <= n; ++j) {
          double p2 = ((2 * j - 1) * t * p1 - (j - 1) * p0) / j;
          p0 = p1;
          p1 = p2;
        }
        dp = n * (t * p1 - p0) / (t * t - 1.0);
        break;
      }
    }
    x[n - 1 - i] = t;
    w[n - 1 - i] = 2.0 / ((1.0 - t * t) * dp * dp);
  }
}
/// Collapsed Duffy rule on the reference triangle (reference inc/quadrature.hpp:61-79).
inline void duffy(int degree, std::vector<double>& px, std::vector<double>& py, std::vector<double>& w) {
  std::vector<double> xu, wu, xv, wv;
  gauss(degree + 1, xu, wu);
  gauss(degree, xv, wv);
  px.clear(); py.clear(); w.clear();
  for (size_t i = 0; i < xu.size(); ++i) {
    double u = 0.5 * (xu[i] + 1.0), a = 0.5 * wu[i];
    for (size_t j = 0; j < xv.size(); ++j) {
      double v = 0.5 * (xv[j] + 1.0), b = 0.5 * wv[j];
      px.push_back(u * (1.0 - v));
      py.push_back(u * v);
      w.push_back(a * b * u);
    }
  }
}

// --------------------------------------------------- small dense Householder
/// Full QR of an m x n row-major matrix A (m >= n not required): returns the
/// m x m orthogonal Q (row-major) and writes R into A.
inline std::vector<double> householder_q(std::vector<double>& A, int m, int n) {
  std::vector<double> Q(size_t(m) * m, 0.0);
  for (int i = 0; i < m; ++i) Q[size_t(i) * m + i] = 1.0;
  const int steps = std::min(m - 1, n);
  std::vector<double> v(m);
  for (int k = 0; k < steps; ++k) {
    double nrm = 0;
    for (int i = k; i < m; ++i) nrm += A[size_t(i) * n + k] * A[size_t(i) * n + k];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    double a0 = A[size_t(k) * n + k];
    double alpha = a0 > 0 ? -nrm : nrm;
    for (int i = 0; i < m; ++i) v[i] = 0;
    v[k] = a0 - alpha;
    for (int i = k + 1; i < m; ++i) v[i] = A[size_t(i) * n + k];
    double vn = 0;
    for (int i = k; i < m; ++i) vn += v[i] * v[i];
    if (vn == 0.0) continue;
    for (int j = 0; j < n; ++j) {  // A <- (I - 2 v v^T / vn) A
      double s = 0;
      for (int i = k; i < m; ++i) s += v[i] * A[size_t(i) * n + j];
      s *= 2.0 / vn;
      for (int i = k; i < m; ++i) A[size_t(i) * n + j] -= s * v[i];
    }
    for (int r = 0; r < m; ++r) {  // Q <- Q (I - 2 v v^T / vn)
      double s = 0;
      for (int i = k; i < m; ++i) s += Q[size_t(r) * m + i] * v[i];
      s *= 2.0 / vn;
      for (int i = k; i < m; ++i) Q[size_t(r) * m + i] -= s * v[i];
    }
  }
  return Q;
}

/// Dense solve with partial pivoting (square, row-major); throws if singular.
inline std::vector<double> dense_solve(std::vector<double> A, std::vector<double> b, int n) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A[size_t(i) * n + k]) > std::abs(A[size_t(p) * n + k])) p = i;
    if (A[size_t(p) * n + k] == 0.0) throw std::runtime_error("singular reference system");
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A[size_t(k) * n + j], A[size_t(p) * n + j]);
      std::swap(b[k], b[p]);
    }
    for (int i = k + 1; i < n; ++i) {
      double l = A[size_t(i) * n + k] / A[size_t(k) * n + k];
      if (l == 0.0) continue;
      for (int j = k; j < n; ++j) A[size_t(i) * n + j] -= l * A[size_t(k) * n + j];
      b[i] -= l * b[k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < n; ++j) s -= A[size_t(i) * n + j] * b[j];
    b[i] = s / A[size_t(i) * n + i];
  }
  return b;
}

// ---------------------------------------------------------------- RT basis
struct RTBasis {
  int k = 0, nfd = 1, n_bubble = 0, n_div = 0, no = 0, nrt = 3;
  std::vector<std::array<Poly, 2>> fn;  // nrt functions: 3*nfd facet, then interior
};

inline RTBasis build_rt_basis(int k) {
  if (k < 0 || k > 6) throw std::invalid_argument("order k must be in 0..6");
  RTBasis B;
  B.k = k;
  B.nfd = k + 1;
  const int ns = Poly::dim(k);
  B.n_div = ns - 1;
  B.no = k * (k + 1);
  B.n_bubble = B.no - B.n_div;
  B.nrt = 3 * B.nfd + B.no;
  std::vector<Poly> q = onb(k);
  std::vector<std::array<Poly, 2>> gen;  // spans RT_k (inc/fespace.hpp:73-86)
  for (const Poly& s : q) {
    gen.push_back({s, Poly::zero(0)});
    gen.push_back({Poly::zero(0), s});
  }
  for (int j = 0; j <= k; ++j) {
    Poly m = Poly::mono(k - j, j);
    gen.push_back({Poly::mono(1, 0).mul(m), Poly::mono(0, 1).mul(m)});
  }
  const int gd = int(gen.size());
  const double vx[3] = {0, 1, 0}, vy[3] = {0, 0, 1};
  // outward reference normals / lengths of edge e = (v[e+1], v[e+2])
  double enx[3], eny[3], elen[3];
  for (int e = 0; e < 3; ++e) {
    double ax = vx[(e + 1) % 3], ay = vy[(e + 1) % 3], bx = vx[(e + 2) % 3], by = vy[(e + 2) % 3];
    elen[e] = std::hypot(bx - ax, by - ay);
    double tx = (bx - ax) / elen[e], ty = (by - ay) / elen[e];
    double nx = ty, ny = -tx;
    if (nx * (ax - vx[e]) + ny * (ay - vy[e]) < 0) { nx = -nx; ny = -ny; }
    enx[e] = nx;
    eny[e] = ny;
  }
  // constraint rows: facet moments (3 nfd), zero-mean divergence moments (n_div)
  const int nm = 3 * B.nfd;
  std::vector<double> M(size_t(nm) * gd, 0.0), D(size_t(std::max(B.n_div, 1)) * gd, 0.0);
  {
    std::vector<double> gx, gw;
    gauss(2 * k + 3, gx, gw);
    double L[8];
    for (int e = 0; e < 3; ++e)
      for (size_t p = 0; p < gx.size(); ++p) {
        double t = gx[p];
        double ax = vx[(e + 1) % 3], ay = vy[(e + 1) % 3], bx = vx[(e + 2) % 3], by = vy[(e + 2) % 3];
        double x = 0.5 * ((1 - t) * ax + (1 + t) * bx), y = 0.5 * ((1 - t) * ay + (1 + t) * by);
        legendre(k, t, L);
        for (int g = 0; g < gd; ++g) {
          double vn = gen[g][0](x, y) * enx[e] + gen[g][1](x, y) * eny[e];
          for (int i = 0; i <= k; ++i) M[size_t(e * B.nfd + i) * gd + g] += 0.5 * (2 * i + 1) * gw[p] * vn * L[i];
        }
      }
    for (int p = 1; p < ns; ++p)
      for (int g = 0; g < gd; ++g) {
        Poly dv = gen[g][0].dx();
        dv.axpy(1.0, gen[g][1].dy());
        D[size_t(p - 1) * gd + g] = l2(dv, q[p]);
      }
  }
  // orthonormal basis W of ker M: trailing columns of Q in M^T = Q R
  std::vector<double> W(size_t(gd) * B.no, 0.0), bub(size_t(gd) * B.n_bubble, 0.0), psi(size_t(gd) * B.n_div, 0.0);
  if (B.no > 0) {
    std::vector<double> Mt(size_t(gd) * nm);
    for (int i = 0; i < nm; ++i)
      for (int g = 0; g < gd; ++g) Mt[size_t(g) * nm + i] = M[size_t(i) * gd + g];
    std::vector<double> Q = householder_q(Mt, gd, nm);
    for (int g = 0; g < gd; ++g)
      for (int j = 0; j < B.no; ++j) W[size_t(g) * B.no + j] = Q[size_t(g) * gd + (nm + j)];
    // DW = D W (n_div x no); (DW)^T = Q2 R2: null space of DW and min-norm preimages
    std::vector<double> DWt(size_t(B.no) * B.n_div, 0.0);
    for (int p = 0; p < B.n_div; ++p)
      for (int j = 0; j < B.no; ++j) {
        double s = 0;
        for (int g = 0; g < gd; ++g) s += D[size_t(p) * gd + g] * W[size_t(g) * B.no + j];
        DWt[size_t(j) * B.n_div + p] = s;
      }
    std::vector<double> R = DWt;
    std::vector<double> Q2 = householder_q(R, B.no, B.n_div);
    for (int p = 0; p < B.n_div; ++p)
      if (std::abs(R[size_t(p) * B.n_div + p]) < 1e-10) throw std::logic_error("interior divergence map is rank-deficient");
    // G-normalised bubbles: W Q2[:, n_div:]
    for (int c = 0; c < B.n_bubble; ++c) {
      std::vector<double> v(gd, 0.0);
      for (int g = 0; g < gd; ++g)
        for (int j = 0; j < B.no; ++j) v[g] += W[size_t(g) * B.no + j] * Q2[size_t(j) * B.no + (B.n_div + c)];
      double nn = 0;
      for (int a = 0; a < gd; ++a)
        for (int b = 0; b < gd; ++b)
          if (v[a] != 0.0 && v[b] != 0.0)
            nn += v[a] * v[b] * (l2(gen[a][0], gen[b][0]) + l2(gen[a][1], gen[b][1]));
      nn = std::sqrt(nn);
      for (int g = 0; g < gd; ++g) bub[size_t(g) * B.n_bubble + c] = v[g] / nn;
    }
    // min-norm y with (DW) y = e_p: y = Q2[:, :n_div] R2^{-T} e_p
    for (int p = 0; p < B.n_div; ++p) {
      std::vector<double> z(B.n_div, 0.0);
      for (int i = 0; i < B.n_div; ++i) {  // R^T z = e_p (forward substitution)
        double s = (i == p) ? 1.0 : 0.0;
        for (int l = 0; l < i; ++l) s -= R[size_t(l) * B.n_div + i] * z[l];
        z[i] = s / R[size_t(i) * B.n_div + i];
      }
      for (int g = 0; g < gd; ++g) {
        double s = 0;
        for (int j = 0; j < B.no; ++j) {
          double y = 0;
          for (int i = 0; i < B.n_div; ++i) y += Q2[size_t(j) * B.no + i] * z[i];
          s += W[size_t(g) * B.no + j] * y;
        }
        psi[size_t(g) * B.n_div + p] = s;
      }
    }
  }
  auto combine = [&](const std::vector<double>& c) {
    std::array<Poly, 2> f = {Poly::zero(0), Poly::zero(0)};
    for (int g = 0; g < gd; ++g)
      if (c[g] != 0.0) {
        f[0].axpy(c[g], gen[g][0]);
        f[1].axpy(c[g], gen[g][1]);
      }
    return f;
  };
  B.fn.resize(B.nrt);
  // facet functions i>=1: [M; D; bub^T G] c = e_(e,i)
  std::vector<double> S(size_t(gd) * gd, 0.0);
  for (int i = 0; i < nm; ++i)
    for (int g = 0; g < gd; ++g) S[size_t(i) * gd + g] = M[size_t(i) * gd + g];
  for (int p = 0; p < B.n_div; ++p)
    for (int g = 0; g < gd; ++g) S[size_t(nm + p) * gd + g] = D[size_t(p) * gd + g];
  for (int c = 0; c < B.n_bubble; ++c)
    for (int g = 0; g < gd; ++g) {
      double s = 0;
      for (int a = 0; a < gd; ++a) {
        double ba = bub[size_t(a) * B.n_bubble + c];
        if (ba != 0.0) s += ba * (l2(gen[a][0], gen[g][0]) + l2(gen[a][1], gen[g][1]));
      }
      S[size_t(nm + B.n_div + c) * gd + g] = s;
    }
  for (int e = 0; e < 3; ++e) {
    std::array<Poly, 2> rt0 = {Poly::mono(1, 0), Poly::mono(0, 1)};
    rt0[0].axpy(-vx[e], Poly::mono(0, 0));
    rt0[1].axpy(-vy[e], Poly::mono(0, 0));
    for (double& t : rt0[0].c) t *= elen[e];
    for (double& t : rt0[1].c) t *= elen[e];
    B.fn[e * B.nfd] = rt0;
    for (int i = 1; i <= k; ++i) {
      std::vector<double> rhs(gd, 0.0);
      rhs[e * B.nfd + i] = 1.0;
      B.fn[e * B.nfd + i] = combine(dense_solve(S, rhs, gd));
    }
  }
  for (int j = 0; j < B.no; ++j) {
    std::vector<double> c(gd);
    for (int g = 0; g < gd; ++g) c[g] = j < B.n_bubble ? bub[size_t(g) * B.n_bubble + j] : psi[size_t(g) * B.n_div + (j - B.n_bubble)];
    B.fn[3 * B.nfd + j] = combine(c);
  }
  return B;
}

/// Reference tensors of one order (see file comment). Index conventions:
///   r in [0, nrt): RT columns (facet (le,i) -> le*nfd+i, interior -> 3nfd+j)
///   m in [0, ns): orthonormal scalar modes
struct RefTensors {
  int k = 0, nfd = 1, nrt = 3, no = 0, ns = 1, nc = 6, nv = 6;
  std::vector<double> G;   // [4][ns][nrt]     sum_q w Jhat_c(q,r) s_m(q)
  std::vector<double> Mm;  // [2][2][nrt][nrt] sum_q w vhat_{r,i} vhat_{s,j}
  std::vector<double> Dv;  // [ns-1][nrt]      sum_q w divhat_r s_m   (m >= 1)
  std::vector<double> Lv;  // [2][nrt]         sum_q w vhat_{r,i}
  std::vector<double> Ev;  // [3][2][ns][nrt]  sum_qe w ehat_{r,l} s_m (edge le)
  std::vector<double> Tv;  // [3][nfd][ns]     sum_qe w L_i(t) s_m   (edge le)
  // volume rule and basis values for pointwise loads: [nq], [nq][2][nrt]
  std::vector<double> qx, qy, qw, vval;
  int nq = 0;
  // pointwise tables for the (trilinear, upwinded) convection form:
  std::vector<double> vjac;  // [nq][4][nrt] reference Jacobians dvx/dx dvx/dy dvy/dx dvy/dy
  std::vector<double> evp;   // [3][nqe][2][nrt] RT values at edge points
  std::vector<double> ew;    // [nqe] edge weights on [-1,1]
  std::vector<double> eleg;  // [nqe][nfd] Legendre L_i(t_q)
  int nqe = 0;
  RTBasis rt;
  std::vector<Poly> scal;
};

inline std::unique_ptr<RefTensors> build_ref_tensors(int k) {
  auto T = std::make_unique<RefTensors>();
  T->rt = build_rt_basis(k);
  const RTBasis& B = T->rt;
  T->k = k;
  T->nfd = B.nfd;
  T->nrt = B.nrt;
  T->no = B.no;
  T->scal = onb(k);
  T->ns = int(T->scal.size());
  T->nc = 6 * B.nfd;
  T->nv = T->nc + B.no;
  const int nrt = B.nrt, ns = T->ns, nfd = B.nfd;
  duffy(3 * k + 4, T->qx, T->qy, T->qw);
  T->nq = int(T->qw.size());
  std::vector<std::array<Poly, 4>> jac(nrt);
  std::vector<Poly> dv(nrt);
  for (int r = 0; r < nrt; ++r) {
    jac[r] = {B.fn[r][0].dx(), B.fn[r][0].dy(), B.fn[r][1].dx(), B.fn[r][1].dy()};
    dv[r] = jac[r][0];
    dv[r].axpy(1.0, jac[r][3]);
  }
  T->G.assign(size_t(4) * ns * nrt, 0.0);
  T->Mm.assign(size_t(4) * nrt * nrt, 0.0);
  T->Dv.assign(size_t(std::max(ns - 1, 1)) * nrt, 0.0);
  T->Lv.assign(size_t(2) * nrt, 0.0);
  T->vval.assign(size_t(T->nq) * 2 * nrt, 0.0);
  std::vector<double> sv(ns), vv(2 * nrt), jv(4 * nrt), dd(nrt);
  for (int q = 0; q < T->nq; ++q) {
    const double x = T->qx[q], y = T->qy[q], w = T->qw[q];
    for (int m = 0; m < ns; ++m) sv[m] = T->scal[m](x, y);
    for (int r = 0; r < nrt; ++r) {
      vv[r] = B.fn[r][0](x, y);
      vv[nrt + r] = B.fn[r][1](x, y);
      for (int c = 0; c < 4; ++c) jv[c * nrt + r] = jac[r][c](x, y);
      dd[r] = dv[r](x, y);
      T->vval[(size_t(q) * 2 + 0) * nrt + r] = vv[r];
      T->vval[(size_t(q) * 2 + 1) * nrt + r] = vv[nrt + r];
    }
    T->vjac.resize(size_t(T->nq) * 4 * nrt);
    for (int c = 0; c < 4; ++c)
      for (int r = 0; r < nrt; ++r) T->vjac[(size_t(q) * 4 + c) * nrt + r] = jv[c * nrt + r];
    for (int c = 0; c < 4; ++c)
      for (int m = 0; m < ns; ++m)
        for (int r = 0; r < nrt; ++r) T->G[(size_t(c) * ns + m) * nrt + r] += w * jv[c * nrt + r] * sv[m];
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j)
        for (int r = 0; r < nrt; ++r)
          for (int s = 0; s < nrt; ++s)
            T->Mm[((size_t(i) * 2 + j) * nrt + r) * nrt + s] += w * vv[i * nrt + r] * vv[j * nrt + s];
    for (int m = 1; m < ns; ++m)
      for (int r = 0; r < nrt; ++r) T->Dv[size_t(m - 1) * nrt + r] += w * dd[r] * sv[m];
    for (int i = 0; i < 2; ++i)
      for (int r = 0; r < nrt; ++r) T->Lv[size_t(i) * nrt + r] += w * vv[i * nrt + r];
  }
  std::vector<double> ex, ew;
  gauss(3 * k + 4, ex, ew);
  T->nqe = int(ex.size());
  T->ew = ew;
  T->eleg.assign(size_t(T->nqe) * nfd, 0.0);
  T->evp.assign(size_t(3) * T->nqe * 2 * nrt, 0.0);
  for (int q = 0; q < T->nqe; ++q) {
    double Lq[8];
    legendre(k, ex[q], Lq);
    for (int i = 0; i < nfd; ++i) T->eleg[size_t(q) * nfd + i] = Lq[i];
  }
  T->Ev.assign(size_t(3) * 2 * ns * nrt, 0.0);
  T->Tv.assign(size_t(3) * nfd * ns, 0.0);
  const double vx[3] = {0, 1, 0}, vy[3] = {0, 0, 1};
  double L[8];
  for (int e = 0; e < 3; ++e)
    for (size_t p = 0; p < ex.size(); ++p) {
      double t = ex[p], w = ew[p];
      double ax = vx[(e + 1) % 3], ay = vy[(e + 1) % 3], bx = vx[(e + 2) % 3], by = vy[(e + 2) % 3];
      double x = 0.5 * ((1 - t) * ax + (1 + t) * bx), y = 0.5 * ((1 - t) * ay + (1 + t) * by);
      for (int m = 0; m < ns; ++m) sv[m] = T->scal[m](x, y);
      legendre(k, t, L);
      for (int l = 0; l < 2; ++l)
        for (int r = 0; r < nrt; ++r) {
          double v = B.fn[r][l](x, y);
          T->evp[((size_t(e) * T->nqe + p) * 2 + l) * nrt + r] = v;
          for (int m = 0; m < ns; ++m) T->Ev[((size_t(e) * 2 + l) * ns + m) * nrt + r] += w * v * sv[m];
        }
      for (int i = 0; i < nfd; ++i)
        for (int m = 0; m < ns; ++m) T->Tv[(size_t(e) * nfd + i) * ns + m] += w * L[i] * sv[m];
    }
  return T;
}

/// Host tables of the element post-processing (reference inc/postprocess.hpp:
/// 24-136), see dev::PostT. The P^{k+1} integrals use the assembly rule (exact
/// for their degree-2k integrands); the error rule is the degree-16 Duffy rule.
struct PostTables {
  int nh = 3, nqe = 0;
  double ref_mean = 0.0;
  std::vector<double> Kh, Bh, ex, ew, eval, ediv, escal, ehi;
};

inline PostTables build_post_tables(const RefTensors& T) {
  PostTables P;
  const std::vector<Poly> hi = onb(T.k + 1);
  const int nh = int(hi.size()), m = nh - 1, ns = T.ns, nrt = T.nrt;
  P.nh = nh;
  P.ref_mean = l2(hi[0], Poly::mono(0, 0));
  std::vector<Poly> a(nh), b(nh);
  for (int s = 0; s < nh; ++s) {
    a[s] = hi[s].dx();
    b[s] = hi[s].dy();
  }
  P.Kh.assign(size_t(3) * m * m, 0.0);
  P.Bh.assign(size_t(2) * m * ns, 0.0);
  std::vector<double> av(nh), bv(nh), sv(ns);
  for (int q = 0; q < T.nq; ++q) {
    const double x = T.qx[q], y = T.qy[q], w = T.qw[q];
    for (int s = 1; s < nh; ++s) {
      av[s] = a[s](x, y);
      bv[s] = b[s](x, y);
    }
    for (int j = 0; j < ns; ++j) sv[j] = T.scal[j](x, y);
    for (int s = 0; s < m; ++s) {
      for (int t = 0; t < m; ++t) {
        const size_t i = size_t(s) * m + t;
        P.Kh[i] += w * av[s + 1] * av[t + 1];
        P.Kh[size_t(m) * m + i] += w * bv[s + 1] * bv[t + 1];
        P.Kh[size_t(2) * m * m + i] += w * (av[s + 1] * bv[t + 1] + bv[s + 1] * av[t + 1]);
      }
      for (int j = 0; j < ns; ++j) {
        P.Bh[size_t(s) * ns + j] += w * av[s + 1] * sv[j];
        P.Bh[size_t(m + s) * ns + j] += w * bv[s + 1] * sv[j];
      }
    }
  }
  std::vector<double> px, py, pw;
  duffy(16, px, py, pw);
  P.nqe = int(pw.size());
  P.ew = pw;
  std::vector<Poly> dv(nrt);
  for (int r = 0; r < nrt; ++r) {
    dv[r] = T.rt.fn[r][0].dx();
    dv[r].axpy(1.0, T.rt.fn[r][1].dy());
  }
  for (int q = 0; q < P.nqe; ++q) {
    const double x = px[q], y = py[q];
    P.ex.push_back(x);
    P.ex.push_back(y);
    for (int l = 0; l < 2; ++l)
      for (int r = 0; r < nrt; ++r) P.eval.push_back(T.rt.fn[r][l](x, y));
    for (int r = 0; r < nrt; ++r) P.ediv.push_back(dv[r](x, y));
    for (int j = 0; j < ns; ++j) P.escal.push_back(T.scal[j](x, y));
    for (int s = 0; s < nh; ++s) P.ehi.push_back(hi[s](x, y));
  }
  return P;
}

}  // namespace host
}  // namespace hpmg
