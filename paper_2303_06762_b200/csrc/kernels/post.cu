// Element-local post-processing and error measurement on the device
// (reference inc/postprocess.hpp:24-188).
//
// postprocess: one thread per element. The reference assembles the P^{k+1}
// stiffness and the gradient-variable load point by point at the assembly
// rule; both integrands are polynomials of degree 2k, so with the reference
// gradients a = d/dx^, b = d/dy^ of the orthonormal P^{k+1} modes they collapse
// to three reference matrices (sum_q w a_s a_t, b_s b_t, a_s b_t + b_s a_t)
// weighted by detJ Ji Ji^T, and two (sum_q w a_s s_m, b_s s_m) contracted with
// Ji and the gradient coefficients. The (ns_hi-1)^2 SPD system is then
// Cholesky-solved in registers/local memory (<= 14 unknowns at k = 3, 35 at
// k = 6; two size classes).
//
// measure_errors: one thread per element over the degree-16 error rule, the
// exact flow evaluated on the device (manufactured / linear) or read from a
// host-tabulated buffer; per-block partials of the four squared norms are
// summed in fixed order by a second one-block kernel (deterministic).
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace hpmg {
namespace dev {

#define HPMG_LAUNCH_CHECK()                                                                        \
  do {                                                                                             \
    cudaError_t err__ = cudaGetLastError();                                                        \
    if (err__ != cudaSuccess) throw std::runtime_error(std::string("CUDA launch (") + __func__ + "): " + cudaGetErrorString(err__)); \
  } while (0)

namespace {

// size classes: k <= 3 (the reference's orders) and k <= 6
constexpr int kMaxH = 35;  // ns_hi - 1 at k = 6
constexpr int kMaxS = 28;  // ns at k = 6

__device__ __forceinline__ void local_coeffs(const PostT& P, const ElemGeo& g, int e, const int* elem_facets,
                                             const double* compound, const double* interior, double* c) {
  const int nfd = P.nfd;
  for (int r = 0; r < P.nrt; ++r) {
    if (r < 3 * nfd) {
      const int le = r / nfd, i = r % nfd;
      const double f = ((i & 1) && g.rho[le] < 0) ? -g.fac[le] : g.fac[le];
      c[r] = f * compound[size_t(elem_facets[e * 3 + le]) * nfd + i];
    } else {
      c[r] = interior[size_t(e) * P.no + (r - 3 * nfd)];
    }
  }
}

template <int MaxRt, int MaxH>
__global__ void k_postprocess(PostT P, const ElemGeo* __restrict__ geo, int ne, const int* __restrict__ elem_facets,
                              double nu, const double* __restrict__ compound, const double* __restrict__ interior,
                              const double* __restrict__ grad, double* __restrict__ post) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const ElemGeo& g = geo[e];
  const int nrt = P.nrt, ns = P.ns, nh = P.nh, m = nh - 1;
  double c[MaxRt];
  local_coeffs(P, g, e, elem_facets, compound, interior, c);
  // mean: sum_q w (J v^ c) / detJ = J (Lv c) / detJ
  double l0 = 0.0, l1 = 0.0;
  for (int r = 0; r < nrt; ++r) {
    l0 = fma(P.Lv[r], c[r], l0);
    l1 = fma(P.Lv[nrt + r], c[r], l1);
  }
  const double um0 = (g.J[0] * l0 + g.J[1] * l1) / g.detJ, um1 = (g.J[2] * l0 + g.J[3] * l1) / g.detJ;
  // physical metric detJ Ji Ji^T (Ji row-major: Ji[0] Ji[1] / Ji[2] Ji[3])
  const double mxx = g.detJ * (g.Ji[0] * g.Ji[0] + g.Ji[1] * g.Ji[1]);
  const double myy = g.detJ * (g.Ji[2] * g.Ji[2] + g.Ji[3] * g.Ji[3]);
  const double mxy = g.detJ * (g.Ji[0] * g.Ji[2] + g.Ji[1] * g.Ji[3]);
  double Lc[MaxH * (MaxH + 1) / 2];  // packed lower Cholesky factor, row-major
  for (int s = 0; s < m; ++s)
    for (int t = 0; t <= s; ++t) {
      const int i = s * m + t;
      Lc[s * (s + 1) / 2 + t] = mxx * P.Kh[i] + myy * P.Kh[m * m + i] + mxy * P.Kh[2 * m * m + i];
    }
  for (int j = 0; j < m; ++j) {
    double d = Lc[j * (j + 1) / 2 + j];
    for (int l = 0; l < j; ++l) d -= Lc[j * (j + 1) / 2 + l] * Lc[j * (j + 1) / 2 + l];
    d = sqrt(d);
    Lc[j * (j + 1) / 2 + j] = d;
    for (int i = j + 1; i < m; ++i) {
      double v = Lc[i * (i + 1) / 2 + j];
      for (int l = 0; l < j; ++l) v -= Lc[i * (i + 1) / 2 + l] * Lc[j * (j + 1) / 2 + l];
      Lc[i * (i + 1) / 2 + j] = v / d;
    }
  }
  const double* G = grad + size_t(e) * 4 * ns;
  double* out = post + size_t(e) * 2 * nh;
  const double sc = -g.detJ / nu;
  for (int comp = 0; comp < 2; ++comp) {
    // rhs_s = -(detJ/nu) sum_m [(Ji00 Ba + Ji10 Bb) G_{comp,x} + (Ji01 Ba + Ji11 Bb) G_{comp,y}]_{s m}
    const double* Gx = G + (2 * comp) * ns;
    const double* Gy = G + (2 * comp + 1) * ns;
    double y[MaxH];
    for (int s = 0; s < m; ++s) {
      double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
      for (int q = 0; q < ns; ++q) {
        const double ba = P.Bh[s * ns + q], bb = P.Bh[(m + s) * ns + q];
        ax = fma(ba, Gx[q], ax);
        ay = fma(ba, Gy[q], ay);
        bx = fma(bb, Gx[q], bx);
        by = fma(bb, Gy[q], by);
      }
      double v = sc * (g.Ji[0] * ax + g.Ji[2] * bx + g.Ji[1] * ay + g.Ji[3] * by);
      for (int l = 0; l < s; ++l) v -= Lc[s * (s + 1) / 2 + l] * y[l];
      y[s] = v / Lc[s * (s + 1) / 2 + s];
    }
    for (int s = m - 1; s >= 0; --s) {
      double v = y[s];
      for (int l = s + 1; l < m; ++l) v -= Lc[l * (l + 1) / 2 + s] * y[l];
      y[s] = v / Lc[s * (s + 1) / 2 + s];
    }
    out[comp * nh] = (comp == 0 ? um0 : um1) / P.ref_mean;
    for (int s = 0; s < m; ++s) out[comp * nh + 1 + s] = y[s];
  }
}

__device__ __forceinline__ double bump(double s) { return s * s * (s - 1.0) * (s - 1.0); }
__device__ __forceinline__ double bump_d1(double s) { return 2.0 * s * (s - 1.0) * (2.0 * s - 1.0); }
__device__ __forceinline__ double bump_d2(double s) { return 12.0 * s * s - 12.0 * s + 2.0; }

/// exact velocity and gradient (row-major d u_i / d x_j) of the named flows
/// (reference inc/manufactured.hpp:21-33, tests/test_postprocess.cpp:120-128)
__device__ __forceinline__ void exact_flow(int kind, double x, double y, double* u, double* gr) {
  if (kind == 1) {
    u[0] = -bump(x) * bump_d1(y);
    u[1] = bump_d1(x) * bump(y);
    gr[0] = -bump_d1(x) * bump_d1(y);
    gr[1] = -bump(x) * bump_d2(y);
    gr[2] = bump_d2(x) * bump(y);
    gr[3] = bump_d1(x) * bump_d1(y);
  } else {
    u[0] = 1 + 2 * y + 3 * x;
    u[1] = 4 - 3 * y + 5 * x;
    gr[0] = 3;
    gr[1] = 2;
    gr[2] = 5;
    gr[3] = -3;
  }
}

constexpr int kErrThreads = 128;

template <int MaxRt>
__global__ void __launch_bounds__(kErrThreads) k_errors(PostT P, const ElemGeo* __restrict__ geo,
                                                        const double* __restrict__ x0, int ne,
                                                        const int* __restrict__ elem_facets, double nu,
                                                        const double* __restrict__ compound,
                                                        const double* __restrict__ interior,
                                                        const double* __restrict__ grad,
                                                        const double* __restrict__ post, int kind,
                                                        const double* __restrict__ ue, const double* __restrict__ ge,
                                                        double* __restrict__ partial) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int nrt = P.nrt, ns = P.ns, nh = P.nh, nq = P.nqe;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
    const ElemGeo& g = geo[e];
    double c[MaxRt];
    local_coeffs(P, g, e, elem_facets, compound, interior, c);
    const double* G = grad + size_t(e) * 4 * ns;
    const double* ps = post + size_t(e) * 2 * nh;
    double su = 0.0, sl = 0.0, sp = 0.0, sd = 0.0;
    for (int q = 0; q < nq; ++q) {
      const double w = P.ew[q] * g.detJ;
      const double xh = P.ex[2 * q], yh = P.ex[2 * q + 1];
      const double* vv = P.eval + size_t(q) * 2 * nrt;
      double h0 = 0.0, h1 = 0.0, dv = 0.0;
      for (int r = 0; r < nrt; ++r) {
        h0 = fma(vv[r], c[r], h0);
        h1 = fma(vv[nrt + r], c[r], h1);
        dv = fma(P.ediv[size_t(q) * nrt + r], c[r], dv);
      }
      const double u0 = (g.J[0] * h0 + g.J[1] * h1) / g.detJ, u1 = (g.J[2] * h0 + g.J[3] * h1) / g.detJ;
      double uex[2], gex[4];
      if (kind == 0) {
        const size_t o = size_t(e) * nq + q;
        uex[0] = ue[2 * o];
        uex[1] = ue[2 * o + 1];
        for (int i = 0; i < 4; ++i) gex[i] = ge[4 * o + i];
      } else {
        const double x = x0[2 * e] + g.J[0] * xh + g.J[1] * yh, y = x0[2 * e + 1] + g.J[2] * xh + g.J[3] * yh;
        exact_flow(kind, x, y, uex, gex);
      }
      su = fma(w, (uex[0] - u0) * (uex[0] - u0) + (uex[1] - u1) * (uex[1] - u1), su);
      const double dd = dv / g.detJ;
      sd = fma(w, dd * dd, sd);
      const double* sv = P.escal + size_t(q) * ns;
      for (int comp = 0; comp < 4; ++comp) {
        double lh = 0.0;
        for (int s = 0; s < ns; ++s) lh = fma(sv[s], G[comp * ns + s], lh);
        const double d = -nu * gex[comp] - lh;
        sl = fma(w, d * d, sl);
      }
      const double* hv = P.ehi + size_t(q) * nh;
      double s0 = 0.0, s1 = 0.0;
      for (int s = 0; s < nh; ++s) {
        s0 = fma(hv[s], ps[s], s0);
        s1 = fma(hv[s], ps[nh + s], s1);
      }
      sp = fma(w, (uex[0] - s0) * (uex[0] - s0) + (uex[1] - s1) * (uex[1] - s1), sp);
    }
    acc[0] += su;
    acc[1] += sl;
    acc[2] += sp;
    acc[3] += sd;
  }
  __shared__ double red[4][kErrThreads];
  for (int j = 0; j < 4; ++j) red[j][threadIdx.x] = acc[j];
  __syncthreads();
  for (int w = kErrThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int j = 0; j < 4; ++j) red[j][threadIdx.x] += red[j][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 4) partial[threadIdx.x * gridDim.x + blockIdx.x] = red[threadIdx.x][0];
}

/// out[j] = sqrt(sum_b partial[j][b]), fixed order
__global__ void k_errors_final(const double* __restrict__ partial, int nblocks, double* __restrict__ out) {
  __shared__ double red[4][32];
  const int j = threadIdx.x / 32, l = threadIdx.x % 32;
  double s = 0.0;
  for (int b = l; b < nblocks; b += 32) s += partial[j * nblocks + b];
  red[j][l] = s;
  __syncthreads();
  if (l == 0) {
    double t = 0.0;
    for (int i = 0; i < 32; ++i) t += red[j][i];
    out[j] = sqrt(t);
  }
}

}  // namespace

void postprocess(const PostT& P, const ElemGeo* geo, int ne, const int* elem_facets, double nu, const double* compound,
                 const double* interior, const double* grad, double* post, cudaStream_t s) {
  if (P.nrt > kMaxRt || P.nh - 1 > kMaxH || P.ns > kMaxS) throw std::runtime_error("order too high for postprocess");
  if (ne == 0) return;
  if (P.nrt <= 24 && P.nh - 1 <= 14)
    k_postprocess<24, 14><<<(ne + 127) / 128, 128, 0, s>>>(P, geo, ne, elem_facets, nu, compound, interior, grad, post);
  else
    k_postprocess<kMaxRt, kMaxH><<<(ne + 127) / 128, 128, 0, s>>>(P, geo, ne, elem_facets, nu, compound, interior,
                                                                   grad, post);
  HPMG_LAUNCH_CHECK();
}

void measure_errors(const PostT& P, const ElemGeo* geo, const double* x0, int ne, const int* elem_facets, double nu,
                    const double* compound, const double* interior, const double* grad, const double* post, int kind,
                    const double* ue, const double* ge, double* partial, double* out4, cudaStream_t s) {
  if (P.nrt > kMaxRt || P.ns > kMaxS) throw std::runtime_error("order too high for measure_errors");
  if (P.nrt <= 24)
    k_errors<24><<<kRedBlocks, kErrThreads, 0, s>>>(P, geo, x0, ne, elem_facets, nu, compound, interior, grad, post,
                                                    kind, ue, ge, partial);
  else
    k_errors<kMaxRt><<<kRedBlocks, kErrThreads, 0, s>>>(P, geo, x0, ne, elem_facets, nu, compound, interior, grad,
                                                        post, kind, ue, ge, partial);
  HPMG_LAUNCH_CHECK();
  k_errors_final<<<1, 128, 0, s>>>(partial, kRedBlocks, out4);
  HPMG_LAUNCH_CHECK();
}

}  // namespace dev
}  // namespace hpmg
