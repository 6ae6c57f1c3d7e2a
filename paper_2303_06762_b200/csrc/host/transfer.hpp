// Host construction of the CR-GMG prolongation between consecutive
// lowest-order levels, in 2x2 blocks (fine free facet x coarse free facet):
//   averaging transfer  (reference inc/transfer.hpp:19-71)
//   interior patches    (inc/transfer.hpp:75-88)
//   harmonic correction P_T = I_T - A_TT^{-1} (A I)_T  (inc/transfer.hpp:95-133)
// The correction reads the assembled fine operator (downloaded once from the
// device). Setup-only work on small fixed-capacity row buffers (a fine row
// touches at most 5 coarse facets, a corrected row at most 9); the apply runs
// on the device (dev::prolong_add / dev::restrict_).
#pragma once

#include <array>
#include <vector>

#include "plan.hpp"

namespace hpmg {
namespace host {

struct BlockCsrH {
  int nrows = 0, ncols = 0;
  std::vector<int> ptr{0}, col;
  std::vector<double> val;  // 4 per block, row-major [t][t']
};

/// 1 - 2 * (barycentric coordinate of the opposite vertex): the CR basis of
/// local facet lf, value 1 at its midpoint (reference inc/cr.hpp:69-77).
inline double cr_basis(const TriMesh& m, int e, int lf, double x, double y) {
  const auto& v = m.ev[e];
  const double px = m.vx[v[lf]], py = m.vy[v[lf]];
  const double ax = m.vx[v[(lf + 1) % 3]], ay = m.vy[v[(lf + 1) % 3]];
  const double bx = m.vx[v[(lf + 2) % 3]], by = m.vy[v[(lf + 2) % 3]];
  const double full = (bx - ax) * (py - ay) - (by - ay) * (px - ax);
  const double part = (bx - ax) * (y - ay) - (by - ay) * (x - ax);
  return 1.0 - 2.0 * part / full;
}

/// Sparse block row with a small fixed capacity, columns kept sorted.
template <int N>
struct BlockRow {
  int n = 0;
  std::array<int, N> col;
  std::array<std::array<double, 4>, N> v;
  std::array<double, 4>& at(int c) {
    int i = 0;
    while (i < n && col[i] < c) ++i;
    if (i < n && col[i] == c) return v[i];
    if (n == N) throw std::runtime_error("transfer row capacity exceeded");
    for (int j = n; j > i; --j) {
      col[j] = col[j - 1];
      v[j] = v[j - 1];
    }
    col[i] = c;
    v[i] = {0.0, 0.0, 0.0, 0.0};
    ++n;
    return v[i];
  }
};

constexpr int kAvgCap = 8;   // fine row of the averaging transfer: <= 5 coarse facets
constexpr int kCorrCap = 16; // corrected row: facets of a coarse element and its neighbours (<= 9)

/// Rows of the averaging transfer (reference inc/transfer.hpp:19-71).
inline std::vector<BlockRow<kAvgCap>> averaging_blocks(const LevelPlan& C, const LevelPlan& F, const Refinement& R) {
  const TriMesh& cm = *C.mesh;
  const TriMesh& fm = *F.mesh;
  std::vector<BlockRow<kAvgCap>> rows(F.nb);
  for (int rf = 0; rf < F.nb; ++rf) {
    const int ff = F.block_facet[rf];
    int se[2] = {-1, -1};
    double sw[2] = {0, 0};
    if (R.fclass[ff] == kMedial) {
      se[0] = R.parent_elem[ff];
      sw[0] = 1.0;
    } else if (R.fclass[ff] == kBoundaryChild) {
      se[0] = cm.fe[R.parent_facet[ff]][0];
      sw[0] = 1.0;
    } else {
      const int pf = R.parent_facet[ff];
      se[0] = cm.fe[pf][0];
      sw[0] = 0.5;
      se[1] = cm.fe[pf][1];
      sw[1] = 0.5;
    }
    double xm, ym, nfx, nfy, tfx, tfy;
    fm.fmid(ff, xm, ym);
    fm.fnormal(ff, nfx, nfy);
    fm.ftan(ff, tfx, tfy);
    for (int s = 0; s < 2; ++s) {
      const int e = se[s];
      if (e < 0) continue;
      for (int i = 0; i < 3; ++i) {
        const int fc = cm.ef[e][i];
        const int cb = C.facet_block[fc];
        if (cb < 0) continue;
        const double phi = sw[s] * cr_basis(cm, e, i, xm, ym);
        double ncx, ncy, tcx, tcy;
        cm.fnormal(fc, ncx, ncy);
        cm.ftan(fc, tcx, tcy);
        auto& b = rows[rf].at(cb);
        b[0] += phi * (nfx * ncx + nfy * ncy);  // (flux, flux)
        b[3] += phi * (tfx * tcx + tfy * tcy);  // (tang, tang)
        b[1] += phi * (nfx * tcx + nfy * tcy);  // (flux, tang)
        b[2] += phi * (tfx * ncx + tfy * ncy);  // (tang, flux)
      }
    }
  }
  return rows;
}

/// Small dense LU solve with partial pivoting, multiple right-hand sides
/// (row-major A n x n, B n x m overwritten by the solution).
inline void lu_solve_multi(std::vector<double> A, int n, std::vector<double>& B, int m) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A[i * n + k]) > std::abs(A[p * n + k])) p = i;
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[p * n + j]);
      for (int j = 0; j < m; ++j) std::swap(B[size_t(k) * m + j], B[size_t(p) * m + j]);
    }
    const double d = A[k * n + k];
    for (int i = k + 1; i < n; ++i) {
      const double l = A[i * n + k] / d;
      if (l == 0.0) continue;
      for (int j = k + 1; j < n; ++j) A[i * n + j] -= l * A[k * n + j];
      for (int j = 0; j < m; ++j) B[size_t(i) * m + j] -= l * B[size_t(k) * m + j];
    }
  }
  for (int j = 0; j < m; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double s = B[size_t(i) * m + j];
      for (int l = i + 1; l < n; ++l) s -= A[i * n + l] * B[size_t(l) * m + j];
      B[size_t(i) * m + j] = s / A[i * n + i];
    }
}

/// Corrected prolongation in block form. `Aval` is the fine level's ELL-BSR
/// value array (bs = 2), pattern from F.cols.
inline BlockCsrH corrected_prolongation(const LevelPlan& C, const LevelPlan& F, const Refinement& R,
                                        const std::vector<double>& Aval) {
  auto rows = averaging_blocks(C, F, R);
  const TriMesh& fm = *F.mesh;
  // interior patches: medial fine facets per coarse element, ascending facet id
  std::vector<std::array<int, 3>> med(R.children.size(), {-1, -1, -1});
  std::vector<int> nmed(R.children.size(), 0);
  for (int ff = 0; ff < fm.nf(); ++ff)
    if (R.fclass[ff] == kMedial && F.facet_block[ff] >= 0) {
      const int e = R.parent_elem[ff];
      med[e][nmed[e]++] = F.facet_block[ff];
    }
  auto Aent = [&](int rb, int rt, int cb, int ct) -> double {
    for (int s = 0; s < kSlots; ++s)
      if (F.cols[size_t(rb) * kSlots + s] == cb) return Aval[((size_t(rb) * kSlots + s) * 2 + rt) * 2 + ct];
    return 0.0;
  };
  std::vector<BlockRow<kCorrCap>> corr(F.nb);
  std::vector<double> Att, B;
  for (size_t e = 0; e < med.size(); ++e) {
    const int nt = 2 * nmed[e];
    if (nt == 0) continue;
    // W_T = (A I_avg) restricted to the rows of T: per T-row, coarse block -> (flux, tang)
    BlockRow<kCorrCap> W[6];
    for (int r = 0; r < nt; ++r) {
      const int rb = med[e][r / 2], rt = r % 2;
      for (int s = 0; s < kSlots; ++s) {
        const int jb = F.cols[size_t(rb) * kSlots + s];
        if (jb < 0) continue;
        for (int jt = 0; jt < 2; ++jt) {
          const double a = Aval[((size_t(rb) * kSlots + s) * 2 + rt) * 2 + jt];
          if (a == 0.0) continue;
          const auto& ar = rows[jb];
          for (int q = 0; q < ar.n; ++q) {
            auto& w = W[r].at(ar.col[q]);
            w[0] += a * ar.v[q][jt * 2 + 0];
            w[1] += a * ar.v[q][jt * 2 + 1];
          }
        }
      }
    }
    BlockRow<kCorrCap> cols;  // union of W columns
    for (int r = 0; r < nt; ++r)
      for (int q = 0; q < W[r].n; ++q) cols.at(W[r].col[q]);
    if (cols.n == 0) continue;
    const int m = 2 * cols.n;
    Att.assign(size_t(nt) * nt, 0.0);
    B.assign(size_t(nt) * m, 0.0);
    for (int r = 0; r < nt; ++r) {
      for (int c = 0; c < nt; ++c) Att[size_t(r) * nt + c] = Aent(med[e][r / 2], r % 2, med[e][c / 2], c % 2);
      for (int q = 0; q < W[r].n; ++q) {
        int j = 0;
        while (cols.col[j] != W[r].col[q]) ++j;
        B[size_t(r) * m + 2 * j] = W[r].v[q][0];
        B[size_t(r) * m + 2 * j + 1] = W[r].v[q][1];
      }
    }
    lu_solve_multi(Att, nt, B, m);
    for (int r = 0; r < nt; ++r)
      for (int j = 0; j < cols.n; ++j) {
        auto& b = corr[med[e][r / 2]].at(cols.col[j]);
        b[(r % 2) * 2 + 0] -= B[size_t(r) * m + 2 * j];
        b[(r % 2) * 2 + 1] -= B[size_t(r) * m + 2 * j + 1];
      }
  }
  BlockCsrH P;
  P.nrows = F.nb;
  P.ncols = C.nb;
  P.col.reserve(size_t(F.nb) * 6);
  P.val.reserve(size_t(F.nb) * 24);
  for (int rf = 0; rf < F.nb; ++rf) {
    BlockRow<kCorrCap> merged;
    for (int q = 0; q < rows[rf].n; ++q) merged.at(rows[rf].col[q]) = rows[rf].v[q];
    for (int q = 0; q < corr[rf].n; ++q) {
      auto& b = merged.at(corr[rf].col[q]);
      for (int t = 0; t < 4; ++t) b[t] += corr[rf].v[q][t];
    }
    for (int q = 0; q < merged.n; ++q) {
      const auto& v = merged.v[q];
      if (v[0] == 0.0 && v[1] == 0.0 && v[2] == 0.0 && v[3] == 0.0) continue;
      P.col.push_back(merged.col[q]);
      for (int t = 0; t < 4; ++t) P.val.push_back(v[t]);
    }
    P.ptr.push_back(int(P.col.size()));
  }
  return P;
}

inline BlockCsrH transpose_blocks(const BlockCsrH& P) {
  BlockCsrH T;
  T.nrows = P.ncols;
  T.ncols = P.nrows;
  std::vector<int> cnt(P.ncols + 1, 0);
  for (int c : P.col) cnt[c + 1]++;
  for (int i = 0; i < P.ncols; ++i) cnt[i + 1] += cnt[i];
  T.ptr = cnt;
  T.col.assign(P.col.size(), 0);
  T.val.assign(P.val.size(), 0.0);
  std::vector<int> pos(cnt.begin(), cnt.end() - 1);
  for (int r = 0; r < P.nrows; ++r)
    for (int q = P.ptr[r]; q < P.ptr[r + 1]; ++q) {
      const int c = P.col[q], d = pos[c]++;
      T.col[d] = r;
      const double* v = &P.val[size_t(q) * 4];
      T.val[size_t(d) * 4 + 0] = v[0];
      T.val[size_t(d) * 4 + 1] = v[2];
      T.val[size_t(d) * 4 + 2] = v[1];
      T.val[size_t(d) * 4 + 3] = v[3];
    }
  return T;
}

}  // namespace host
}  // namespace hpmg
