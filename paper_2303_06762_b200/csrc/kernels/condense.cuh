// Element-local assembly + static condensation (reference
// inc/assembly.hpp:205-364, build_local_blocks + condense_local), written as a
// cooperative routine over (tid, nthr) so one CTA condenses one element.
//
// Affine elements let every Stokes-type integral factor as
//   (reference tensor, tabulated once per k)  x  (J, J^-1, orientation),
// see host/basis.hpp. Per element this kernel only performs small dense
// contractions; the dominant work is the (nu/detJ) C^T C product and the
// elimination of nz = k(k+1) + ns-1 interior unknowns, i.e. FP64 FMA-bound.
//
// The same source compiles for the host (HPMG_HOST_EMUL) with tid=0, nthr=1
// and SYNC() a no-op; tests/native uses that build to check the arithmetic
// against the CPU oracle without a GPU. The product only launches the kernel.
#pragma once

#include <cmath>

#ifndef HPMG_HD
#ifdef __CUDACC__
#define HPMG_HD __host__ __device__
#define HPMG_D __device__
#else
#define HPMG_D
#define HPMG_HD
#endif
#endif

namespace hpmg {

/// Per-order reference tensors (device pointers or host pointers in emulation).
struct RefT {
  int k, nfd, nrt, no, ns, nc, nv;
  const double* G;   // [4][ns][nrt]
  const double* Mm;  // [4][nrt][nrt]
  const double* Dv;  // [ns-1][nrt]
  const double* Lv;  // [2][nrt]
  const double* Ev;  // [3][2][ns][nrt]
  const double* Tv;  // [3][nfd][ns]
  const double* vval;  // [nq][2][nrt] (pointwise loads)
  const double* qw;    // [nq]
  int nq;
  // convection (Oseen) tables
  const double* vjac;  // [nq][4][nrt]
  const double* evp;   // [3][nqe][2][nrt]
  const double* ew;    // [nqe]
  const double* eleg;  // [nqe][nfd]
  int nqe;
};

/// Wind tables of one element (scratch): physical wind at the volume nodes,
/// and per edge node the normal wind w.n_out and (Newton) the upwind trace
/// vector: the RT trace of the wind on outflow nodes, its tangential skeleton
/// trace on inflow nodes (reference inc/assembly.hpp:300-321).
struct WindTab {
  const double* wq = nullptr;  // [nq][2]
  const double* wn = nullptr;  // [3][nqe]
  const double* up = nullptr;  // [3][nqe][2]
  int newton = 0;
};

/// Physical Jacobian (row-major g0..g3) of RT local function r at volume node q.
template <class Geo>
HPMG_HD inline void rt_grad(const RefT& T, const Geo& g, const double* fr, int q, int r, double* gr) {
  const int nrt = T.nrt;
  const double* vj = T.vjac + size_t(q) * 4 * nrt;
  const double h00 = vj[r], h01 = vj[nrt + r], h10 = vj[2 * nrt + r], h11 = vj[3 * nrt + r];
  const double t00 = g.J[0] * h00 + g.J[1] * h10, t01 = g.J[0] * h01 + g.J[1] * h11;
  const double t10 = g.J[2] * h00 + g.J[3] * h10, t11 = g.J[2] * h01 + g.J[3] * h11;
  const double gs = fr[r] / g.detJ;
  gr[0] = (t00 * g.Ji[0] + t01 * g.Ji[2]) * gs;
  gr[1] = (t00 * g.Ji[1] + t01 * g.Ji[3]) * gs;
  gr[2] = (t10 * g.Ji[0] + t11 * g.Ji[2]) * gs;
  gr[3] = (t10 * g.Ji[1] + t11 * g.Ji[3]) * gs;
}

/// Test-function trace difference D on edge le at edge node q (RT column:
/// T - (T.n)n; tangential column of this edge: -T; else zero). False if zero.
template <class Geo>
HPMG_HD inline bool test_trace(const RefT& T, const Geo& g, const double* fr, int le, int q, int a, double* ta) {
  const int nfd = T.nfd, nc = T.nc, nrt = T.nrt;
  const bool ra = a < 3 * nfd || a >= nc;
  if (ra) {
    const int r = a < 3 * nfd ? a : 3 * nfd + (a - nc);
    const double* ev = T.evp + size_t(le * T.nqe + q) * 2 * nrt;
    const double e0 = ev[r], e1 = ev[nrt + r], f = fr[r] / g.detJ;
    const double T0 = (g.J[0] * e0 + g.J[1] * e1) * f, T1 = (g.J[2] * e0 + g.J[3] * e1) * f;
    const double nx = g.n[2 * le], ny = g.n[2 * le + 1];
    const double tn = T0 * nx + T1 * ny;
    ta[0] = T0 - tn * nx;
    ta[1] = T1 - tn * ny;
    return true;
  }
  if ((a - 3 * nfd) / nfd != le) return false;
  const int i = (a - 3 * nfd) % nfd;
  double lg = T.eleg[q * nfd + i];
  if (g.rho[le] < 0 && (i & 1)) lg = -lg;
  ta[0] = -lg * g.tf[2 * le];
  ta[1] = -lg * g.tf[2 * le + 1];
  return true;
}

/// Convection entry A(a, b) of the upwinded transport form linearised about
/// the wind (reference inc/assembly.hpp:254-275 volume, :294-321 facets;
/// Picard, plus the Newton terms :265-273, :322-328 when W.newton). Evaluated
/// pointwise: the upwind switch depends on the sign of w.n at every edge node.
template <class Geo>
HPMG_HD inline double convection_entry(const RefT& T, const Geo& g, const double* fr, const WindTab& W, int a,
                                       int b) {
  const int nfd = T.nfd, nc = T.nc, nrt = T.nrt;
  const bool ra = a < 3 * nfd || a >= nc, rb = b < 3 * nfd || b >= nc;
  const int r = ra ? (a < 3 * nfd ? a : 3 * nfd + (a - nc)) : -1;
  const int s = rb ? (b < 3 * nfd ? b : 3 * nfd + (b - nc)) : -1;
  double acc = 0.0;
  const double J0 = g.J[0], J1 = g.J[1], J2 = g.J[2], J3 = g.J[3];
  // volume: -(u (x) w, grad v) [Picard] - (w (x) u, grad v) [Newton], test r, trial s
  if (ra && rb) {
    for (int q = 0; q < T.nq; ++q) {
      const double* vv = T.vval + size_t(q) * 2 * nrt;
      double gr[4];
      rt_grad(T, g, fr, q, r, gr);
      const double vs = fr[s] / g.detJ;
      const double v0 = (J0 * vv[s] + J1 * vv[nrt + s]) * vs, v1 = (J2 * vv[s] + J3 * vv[nrt + s]) * vs;
      const double wx = W.wq[2 * q], wy = W.wq[2 * q + 1];
      const double w = T.qw[q] * g.detJ;
      acc -= w * (v0 * (gr[0] * wx + gr[1] * wy) + v1 * (gr[2] * wx + gr[3] * wy));
      if (W.newton) acc -= w * (wx * (gr[0] * v0 + gr[1] * v1) + wy * (gr[2] * v0 + gr[3] * v1));
    }
  }
  // facets: upwinded transport of the trace, tested with the tangential difference
  for (int le = 0; le < 3; ++le) {
    const double nx = g.n[2 * le], ny = g.n[2 * le + 1];
    const bool at = !ra && (a - 3 * nfd) / nfd == le;
    if (!ra && !at) continue;
    const bool bt = !rb && (b - 3 * nfd) / nfd == le;
    const bool newton_col = W.newton && b < 3 * nfd;  // Newton couples the flux trial columns
    if (!rb && !bt && !newton_col) continue;
    for (int q = 0; q < T.nqe; ++q) {
      const double wnq = W.wn[le * T.nqe + q];
      double ta[2];
      test_trace(T, g, fr, le, q, a, ta);
      const double* ev = T.evp + size_t(le * T.nqe + q) * 2 * nrt;
      double tb0 = 0.0, tb1 = 0.0;
      if (rb) {
        const double e0 = ev[s], e1 = ev[nrt + s], f = fr[s] / g.detJ;
        tb0 = (J0 * e0 + J1 * e1) * f;
        tb1 = (J2 * e0 + J3 * e1) * f;
      } else if (bt) {
        const int i = (b - 3 * nfd) % nfd;
        double lg = T.eleg[q * nfd + i];
        if (g.rho[le] < 0 && (i & 1)) lg = -lg;
        tb0 = lg * g.tf[2 * le];
        tb1 = lg * g.tf[2 * le + 1];
      }
      const double wds = T.ew[q] * g.ds[le];
      // Picard: outflow couples RT trial columns, inflow tangential ones
      if (wnq != 0.0 && (rb || bt) && (wnq > 0) == rb) acc += wds * wnq * (ta[0] * tb0 + ta[1] * tb1);
      if (newton_col) {
        const double tup = ta[0] * W.up[2 * (le * T.nqe + q)] + ta[1] * W.up[2 * (le * T.nqe + q) + 1];
        if (tup != 0.0) acc += wds * tup * (tb0 * nx + tb1 * ny);
      }
    }
  }
  return acc;
}

/// Newton load of test column a: -(w (x) w, grad v) + <w.n (w_up . D(v))>
/// (reference inc/assembly.hpp:273, :327).
template <class Geo>
HPMG_HD inline double newton_rhs(const RefT& T, const Geo& g, const double* fr, const WindTab& W, int a) {
  const int nfd = T.nfd, nc = T.nc;
  const bool ra = a < 3 * nfd || a >= nc;
  double acc = 0.0;
  if (ra) {
    const int r = a < 3 * nfd ? a : 3 * nfd + (a - nc);
    for (int q = 0; q < T.nq; ++q) {
      double gr[4];
      rt_grad(T, g, fr, q, r, gr);
      const double wx = W.wq[2 * q], wy = W.wq[2 * q + 1];
      acc -= T.qw[q] * g.detJ * (wx * (gr[0] * wx + gr[1] * wy) + wy * (gr[2] * wx + gr[3] * wy));
    }
  }
  for (int le = 0; le < 3; ++le)
    for (int q = 0; q < T.nqe; ++q) {
      double ta[2];
      if (!test_trace(T, g, fr, le, q, a, ta)) break;
      const int e = le * T.nqe + q;
      const double tup = ta[0] * W.up[2 * e] + ta[1] * W.up[2 * e + 1];
      acc += T.ew[q] * g.ds[le] * W.wn[e] * tup;
    }
  return acc;
}

/// Per-element geometry, 32 doubles (packed on the host).
struct ElemGeo {
  double J[4];      // J00 J01 J10 J11 (columns: v1-v0, v2-v0)
  double Ji[4];     // inverse
  double detJ;
  double fac[3];    // sigma |F| / |ref edge|
  double rho[3];    // +1 / -1 (local edge direction vs global)
  double n[6];      // outward unit normal per local edge
  double tf[6];     // global unit tangent per local facet
  double ds[3];     // |F| / 2
};

struct CondenseParams {
  double nu, mass;        // mass = beta + mass_coef
  int load_mode;          // 0 none, 1 constant per element, 2 pointwise [nq][2]
  int newton;             // Newton linearisation about the wind (needs the wind)
  double mass_coef;       // pseudo-time coefficient multiplying the mass field load
};

/// Scratch layout (doubles): C[4ns*nv] A[nv*nv] P[(ns-1)*nv] rhs[nv] aug[nz*(nz+nc+1)] fac[nrt]
/// + the tables wq[2nq] wn[3nqe] up[6nqe] mq[2nq].
HPMG_HD inline int condense_scratch(int ns, int nv, int nc, int nz, int nrt, int nq, int nqe) {
  return 4 * ns * nv + nv * nv + (ns > 1 ? (ns - 1) * nv : 0) + nv + nz * (nz + nc + 1) + nrt + 8 + 4 * nq +
         9 * nqe + 8;
}

#ifndef SYNC
#define SYNC() __syncthreads()
#endif

/// Computes the condensed element matrix Ac (nc x nc, row-major, reference
/// local order: 3 nfd flux, 3 nfd tangential) and load vector rc (nc).
/// Recovery mode (reference recover_locals, inc/assembly.hpp:513-549): with
/// xc != nullptr the element's skeleton coefficients are given and, instead of
/// Ac / rc, z = M_zz^{-1}(r_z - M_zc xc) (interior RT coefficients then the
/// zero-mean pressure modes) goes to zout and the gradient variable
/// -(nu/detJ) C [xc; z_interior] to gout.
HPMG_D inline void condense_element(int tid, int nthr, const RefT& T, const ElemGeo& g, const CondenseParams& prm,
                                     const double* load, double* scratch, double* Ac, double* rc,
                                     const double* xc = nullptr, double* zout = nullptr, double* gout = nullptr,
                                     const double* xw = nullptr, const double* xm = nullptr) {
  const int ns = T.ns, nv = T.nv, nc = T.nc, nrt = T.nrt, nfd = T.nfd, no = T.no;
  const int np = ns - 1, nz = no + np, nC = 4 * ns;
  double* C = scratch;
  double* A = C + nC * nv;
  double* P = A + nv * nv;
  double* rhs = P + (np > 0 ? np * nv : 0);
  double* aug = rhs + nv;
  double* fr = aug + nz * (nz + nc + 1);  // orientation factor per RT column
  double* wq = fr + nrt + 8;               // [nq][2] physical wind at the volume nodes
  double* wn = wq + 2 * T.nq;              // [3][nqe] w.n_out at the edge nodes
  double* up = wn + 3 * T.nqe;             // [3][nqe][2] upwind wind trace (Newton)
  double* mq = up + 6 * T.nqe;             // [nq][2] physical mass field (pseudo-time load)
  const int naug = nz + nc + 1;
  WindTab W;
  W.wq = wq;
  W.wn = wn;
  W.up = up;
  W.newton = xw ? prm.newton : 0;

  for (int r = tid; r < nrt; r += nthr) {
    if (r < 3 * nfd) {
      int le = r / nfd, i = r % nfd;
      double f = g.fac[le];
      fr[r] = ((i & 1) && g.rho[le] < 0) ? -f : f;
    } else {
      fr[r] = 1.0;
    }
  }
  SYNC();
  if (xw) {
    // wind in the RT part of the local basis: wrt[r] = xw[vel_of_rt(r)]
    for (int q = tid; q < T.nq; q += nthr) {
      double sx = 0.0, sy = 0.0;
      for (int r = 0; r < nrt; ++r) {
        const double c = xw[r < 3 * nfd ? r : nc + (r - 3 * nfd)] * fr[r] / g.detJ;
        const double v0 = T.vval[(q * 2) * nrt + r], v1 = T.vval[(q * 2 + 1) * nrt + r];
        sx += c * (g.J[0] * v0 + g.J[1] * v1);
        sy += c * (g.J[2] * v0 + g.J[3] * v1);
      }
      wq[2 * q] = sx;
      wq[2 * q + 1] = sy;
    }
    for (int e = tid; e < 3 * T.nqe; e += nthr) {
      const int le = e / T.nqe, q = e % T.nqe;
      const double* ev = T.evp + size_t(le * T.nqe + q) * 2 * nrt;
      double sx = 0.0, sy = 0.0, sabs = 0.0;
      for (int r = 0; r < nrt; ++r) {
        const double c = xw[r < 3 * nfd ? r : nc + (r - 3 * nfd)] * fr[r] / g.detJ;
        const double tx = g.J[0] * ev[r] + g.J[1] * ev[nrt + r], ty = g.J[2] * ev[r] + g.J[3] * ev[nrt + r];
        sx += c * tx;
        sy += c * ty;
        sabs += fabs(c) * sqrt(tx * tx + ty * ty);
      }
      // w.n_out, and the tangential skeleton trace of the wind on this edge
      double lt = 0.0;
      for (int i = 0; i < nfd; ++i) {
        double lg = T.eleg[q * nfd + i];
        if (g.rho[le] < 0 && (i & 1)) lg = -lg;
        lt += xw[3 * nfd + le * nfd + i] * lg;
      }
      // A wind tangential to the edge (no-slip walls, the lid, a solenoidal
      // field along the boundary, a node where it vanishes) has w.n = 0 in
      // exact arithmetic but a round-off sign from the basis tables; the
      // reference's upwind switch (w.n > 0, assembly.hpp:316) would pick the
      // Newton upwind trace by that sign. |w.n| below 1e-13 of the magnitude
      // of the terms it is summed from (plus the tangential trace) counts as
      // the exact zero (inflow branch), in the oracle as well.
      double wne = sx * g.n[2 * le] + sy * g.n[2 * le + 1];
      if (fabs(wne) <= 1e-13 * (sabs + fabs(lt))) wne = 0.0;
      wn[e] = wne;
      if (wne > 0) {
        up[2 * e] = sx;
        up[2 * e + 1] = sy;
      } else {  // inflow: the tangential skeleton trace
        up[2 * e] = lt * g.tf[2 * le];
        up[2 * e + 1] = lt * g.tf[2 * le + 1];
      }
    }
  }
  if (xm) {
    // pseudo-time mass field, physical values at the volume nodes
    for (int q = tid; q < T.nq; q += nthr) {
      double sx = 0.0, sy = 0.0;
      for (int r = 0; r < nrt; ++r) {
        const double c = xm[r < 3 * nfd ? r : nc + (r - 3 * nfd)] * fr[r] / g.detJ;
        const double v0 = T.vval[(q * 2) * nrt + r], v1 = T.vval[(q * 2 + 1) * nrt + r];
        sx += c * (g.J[0] * v0 + g.J[1] * v1);
        sy += c * (g.J[2] * v0 + g.J[3] * v1);
      }
      mq[2 * q] = sx;
      mq[2 * q + 1] = sy;
    }
  }
  SYNC();
  // ---- gradient coupling C (4ns x nv) and divergence moments P ----
  for (int e = tid; e < nC * nv; e += nthr) {
    const int row = e / nv, a = e % nv;
    const int c = row / ns, m = row % ns, c0 = c >> 1, c1 = c & 1;
    double s = 0.0;
    if (a < 3 * nfd || a >= nc) {
      const int r = a < 3 * nfd ? a : 3 * nfd + (a - nc);
      // volume: fr * sum_ij J[c0][i] Ji[j][c1] G[2i+j][m][r]
      double vol = 0.0;
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
          vol += g.J[c0 * 2 + i] * g.Ji[j * 2 + c1] * T.G[((2 * i + j) * ns + m) * nrt + r];
      // edges: -ds n_j fr/detJ sum_k Pi[c0][k] sum_l J[k][l] E[le][l][m][r]
      double edg = 0.0;
      for (int le = 0; le < 3; ++le) {
        const double nx = g.n[2 * le], ny = g.n[2 * le + 1];
        const double e0 = T.Ev[((le * 2 + 0) * ns + m) * nrt + r], e1 = T.Ev[((le * 2 + 1) * ns + m) * nrt + r];
        const double t0 = g.J[0] * e0 + g.J[1] * e1, t1 = g.J[2] * e0 + g.J[3] * e1;  // J ehat
        const double tn = t0 * nx + t1 * ny;
        const double d = (c0 == 0 ? t0 - tn * nx : t1 - tn * ny);
        edg += g.ds[le] * (c1 == 0 ? nx : ny) * d;
      }
      s = fr[r] * vol - fr[r] / g.detJ * edg;
    } else {
      // tangential column (le, p): + ds sgn tf[c0] n[c1] Tv[le][p][m]
      const int le = (a - 3 * nfd) / nfd, p = (a - 3 * nfd) % nfd;
      const double sg = ((p & 1) && g.rho[le] < 0) ? -1.0 : 1.0;
      s = g.ds[le] * sg * g.tf[2 * le + c0] * g.n[2 * le + c1] * T.Tv[(le * nfd + p) * ns + m];
    }
    C[row * nv + a] = s;
  }
  for (int e = tid; e < np * nv; e += nthr) {
    const int m = e / nv, a = e % nv;
    double s = 0.0;
    if (a < 3 * nfd || a >= nc) {
      const int r = a < 3 * nfd ? a : 3 * nfd + (a - nc);
      s = fr[r] * T.Dv[m * nrt + r];
    }
    P[m * nv + a] = s;
  }
  for (int a = tid; a < nv; a += nthr) {
    double s = 0.0;
    if (prm.load_mode != 0 && (a < 3 * nfd || a >= nc)) {
      const int r = a < 3 * nfd ? a : 3 * nfd + (a - nc);
      if (prm.load_mode == 1) {
        const double jf0 = load[0] * g.J[0] + load[1] * g.J[2], jf1 = load[0] * g.J[1] + load[1] * g.J[3];
        s = fr[r] * (jf0 * T.Lv[r] + jf1 * T.Lv[nrt + r]);
      } else {
        for (int q = 0; q < T.nq; ++q) {
          const double fx = load[2 * q], fy = load[2 * q + 1];
          const double jf0 = fx * g.J[0] + fy * g.J[2], jf1 = fx * g.J[1] + fy * g.J[3];
          s += T.qw[q] * (jf0 * T.vval[(q * 2) * nrt + r] + jf1 * T.vval[(q * 2 + 1) * nrt + r]);
        }
        s *= fr[r];
      }
    }
    if (xm && (a < 3 * nfd || a >= nc)) {
      // + mass_coef (m_prev, v): backward-Euler pseudo-time load (reference assembly.hpp:273-276)
      const int r = a < 3 * nfd ? a : 3 * nfd + (a - nc);
      double sm = 0.0;
      for (int q = 0; q < T.nq; ++q) {
        const double fx = mq[2 * q], fy = mq[2 * q + 1];
        const double jf0 = fx * g.J[0] + fy * g.J[2], jf1 = fx * g.J[1] + fy * g.J[3];
        sm += T.qw[q] * (jf0 * T.vval[(q * 2) * nrt + r] + jf1 * T.vval[(q * 2 + 1) * nrt + r]);
      }
      s += prm.mass_coef * fr[r] * sm;
    }
    if (W.newton) s += newton_rhs(T, g, fr, W, a);
    rhs[a] = s;
  }
  SYNC();
  // ---- A = mass part + (nu/detJ) C^T C ----
  const double JtJ[4] = {g.J[0] * g.J[0] + g.J[2] * g.J[2], g.J[0] * g.J[1] + g.J[2] * g.J[3],
                         g.J[1] * g.J[0] + g.J[3] * g.J[2], g.J[1] * g.J[1] + g.J[3] * g.J[3]};
  const double visc = prm.nu / g.detJ;
  for (int e = tid; e < nv * nv; e += nthr) {
    const int a = e / nv, b = e % nv;
    double m = 0.0;
    const bool ra = a < 3 * nfd || a >= nc, rb = b < 3 * nfd || b >= nc;
    if (prm.mass != 0.0 && ra && rb) {
      const int r = a < 3 * nfd ? a : 3 * nfd + (a - nc), s = b < 3 * nfd ? b : 3 * nfd + (b - nc);
      double acc = 0.0;
      for (int ij = 0; ij < 4; ++ij) acc += JtJ[ij] * T.Mm[(ij * nrt + r) * nrt + s];
      m = prm.mass * fr[r] * fr[s] / g.detJ * acc;
    }
    double cc = 0.0;
    for (int row = 0; row < nC; ++row) cc += C[row * nv + a] * C[row * nv + b];
    A[e] = m + visc * cc + (xw ? convection_entry(T, g, fr, W, a, b) : 0.0);
  }
  SYNC();
  if (nz == 0) {
    if (xc) {
      for (int row = tid; row < nC; row += nthr) {
        double s = 0.0;
        for (int a = 0; a < nc; ++a) s += C[row * nv + a] * xc[a];
        gout[row] = -visc * s;
      }
      return;
    }
    for (int e = tid; e < nc * nc; e += nthr) Ac[e] = A[(e / nc) * nv + (e % nc)];
    for (int a = tid; a < nc; a += nthr) rc[a] = rhs[a];
    return;
  }
  // ---- eliminate z = (interior velocity, zero-mean pressure) ----
  // aug = [Mzz | Mzc | rz], Mzz = [[A_oo, -P_o^T], [-P_o, 0]], Mzc = [A_oc; -P_c]
  for (int e = tid; e < nz * naug; e += nthr) {
    const int i = e / naug, j = e % naug;
    double v = 0.0;
    if (j < nz) {
      if (i < no && j < no) v = A[(nc + i) * nv + nc + j];
      else if (i < no) v = -P[(j - no) * nv + nc + i];
      else if (j < no) v = -P[(i - no) * nv + nc + j];
    } else if (j < nz + nc) {
      const int cidx = j - nz;
      v = i < no ? A[(nc + i) * nv + cidx] : -P[(i - no) * nv + cidx];
    } else {
      v = i < no ? rhs[nc + i] : 0.0;
    }
    aug[e] = v;
  }
  SYNC();
  // Gaussian elimination with partial pivoting (pivot search by every thread
  // redundantly: nz <= 21, so the search is cheaper than a reduction)
  for (int kk = 0; kk < nz; ++kk) {
    int piv = kk;
    double best = aug[kk * naug + kk] < 0 ? -aug[kk * naug + kk] : aug[kk * naug + kk];
    for (int i = kk + 1; i < nz; ++i) {
      double v = aug[i * naug + kk];
      v = v < 0 ? -v : v;
      if (v > best) { best = v; piv = i; }
    }
    SYNC();
    if (piv != kk)
      for (int j = tid; j < naug; j += nthr) {
        double t = aug[kk * naug + j];
        aug[kk * naug + j] = aug[piv * naug + j];
        aug[piv * naug + j] = t;
      }
    SYNC();
    const double inv = 1.0 / aug[kk * naug + kk];
    for (int e = tid; e < (nz - kk - 1) * (naug - kk - 1); e += nthr) {
      const int i = kk + 1 + e / (naug - kk - 1), j = kk + 1 + e % (naug - kk - 1);
      aug[i * naug + j] -= aug[i * naug + kk] * inv * aug[kk * naug + j];
    }
    SYNC();
  }
  // back substitution on the nc + 1 right-hand sides (column-parallel)
  for (int j = nz + tid; j < naug; j += nthr) {
    for (int i = nz - 1; i >= 0; --i) {
      double s = aug[i * naug + j];
      for (int l = i + 1; l < nz; ++l) s -= aug[i * naug + l] * aug[l * naug + j];
      aug[i * naug + j] = s / aug[i * naug + i];
    }
  }
  SYNC();
  if (xc) {
    // z = y - X xc, xv = [xc; z_interior] staged in rhs[], then L = -(nu/detJ) C xv
    for (int i = tid; i < nz; i += nthr) {
      double s = aug[i * naug + nz + nc];
      for (int j = 0; j < nc; ++j) s -= aug[i * naug + nz + j] * xc[j];
      zout[i] = s;
      if (i < no) rhs[nc + i] = s;
    }
    for (int a = tid; a < nc; a += nthr) rhs[a] = xc[a];
    SYNC();
    for (int row = tid; row < nC; row += nthr) {
      double s = 0.0;
      for (int a = 0; a < nv; ++a) s += C[row * nv + a] * rhs[a];
      gout[row] = -visc * s;
    }
    return;
  }
  // Ac = A_cc - Mcz X, rc = r_c - Mcz y with Mcz = [A_co, -P_c^T]
  for (int e = tid; e < nc * (nc + 1); e += nthr) {
    const int a = e / (nc + 1), j = e % (nc + 1);
    double s = 0.0;
    for (int i = 0; i < no; ++i) s += A[a * nv + nc + i] * aug[i * naug + nz + j];
    for (int m = 0; m < np; ++m) s -= P[m * nv + a] * aug[(no + m) * naug + nz + j];
    if (j < nc) Ac[a * nc + j] = A[a * nv + j] - s;
    else rc[a] = rhs[a] - s;
  }
}

}  // namespace hpmg
