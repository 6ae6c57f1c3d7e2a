// Structure of the CR-GMG prolongation between consecutive lowest-order
// levels, in 2x2 blocks (fine free facet x coarse free facet):
//   averaging transfer  (reference inc/transfer.hpp:19-71), geometry only
//   interior patches    (inc/transfer.hpp:75-88)
//   the pattern of the harmonic correction P_T = I_T - A_TT^{-1} (A I)_T
//   (inc/transfer.hpp:95-133), whose values the device computes from the
//   current fine operator (kernels.cu corrected_prolongation).
// Setup-only host work on small fixed-capacity row buffers (a fine row
// touches at most 5 coarse facets, a corrected row at most 9).
#pragma once

#include <algorithm>
#include <climits>
#include <new>
#include <array>
#include <memory>
#include <utility>
#include <thread>
#include <vector>

#include "plan.hpp"

namespace hpmg {
namespace host {

struct BlockCsrH {
  int nrows = 0, ncols = 0;
  std::vector<int> ptr{0};
  BigVec<int> col;
  BigVec<double> val;  // 4 per block, row-major [t][t']
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

/// Array of n default-constructed T whose pages are first touched by
/// parallel_for threads (a serial std::vector<T>(n) of ~100 MB of row
/// buffers spends most of its time in page faults). T trivially destructible.
template <class T>
struct ParArray {
  T* p = nullptr;
  int n = 0;
  explicit ParArray(int count) : p(static_cast<T*>(::operator new(sizeof(T) * size_t(std::max(count, 1))))), n(count) {
    parallel_for(n, [&](int i) { new (p + i) T(); });
  }
  ParArray(const ParArray&) = delete;
  ParArray& operator=(const ParArray&) = delete;
  ParArray(ParArray&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  ~ParArray() { ::operator delete(p); }
  T& operator[](int i) { return p[i]; }
  const T& operator[](int i) const { return p[i]; }
};

/// Sorted set of at most N block columns (no values).
template <int N>
struct ColRow {
  int n = 0;
  int col[N];
  void add(int c) {
    int i = 0;
    while (i < n && col[i] < c) ++i;
    if (i < n && col[i] == c) return;
    if (n == N) throw std::runtime_error("transfer row capacity exceeded");
    for (int j = n; j > i; --j) col[j] = col[j - 1];
    col[i] = c;
    ++n;
  }
};

constexpr int kAvgCap = 8;   // fine row of the averaging transfer: <= 5 coarse facets
constexpr int kCorrCap = 16; // corrected row: facets of a coarse element and its neighbours (<= 9)

/// Rows of the averaging transfer (reference inc/transfer.hpp:19-71).
inline ParArray<BlockRow<kAvgCap>> averaging_blocks(const LevelPlan& C, const LevelPlan& F, const Refinement& R) {
  const TriMesh& cm = *C.mesh;
  const TriMesh& fm = *F.mesh;
  ParArray<BlockRow<kAvgCap>> rows(F.nb);
  parallel_for(F.nb, [&](int rf) {
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
  });
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

/// Structure of the corrected prolongation for the device build (built once
/// per level pair; only A changes between linearisations): the averaging
/// transfer as block CSR (geometry only), per coarse element its interior
/// (medial) fine blocks and the coarse columns their correction touches, the
/// final pattern P = averaging + correction (zero blocks kept, so the pattern
/// never depends on values) with the averaging values as its base, and the
/// block positions where each element's correction lands.
struct TransferPlan {
  static constexpr int kMedMax = 3, kColMax = kCorrCap;
  int nrows = 0, ncols = 0, nelem = 0;
  BlockCsrH avg;                      // fine rows of the averaging transfer
  BlockCsrH P;                        // final pattern (values built on the device)
  std::vector<int> nmed, med;         // [nelem], [nelem][3] fine blocks (ascending facet id)
  std::vector<int> ncol, col;         // [nelem], [nelem][kColMax] coarse blocks (ascending)
  std::vector<int> pos;               // [nelem][3][kColMax] block index into P (or -1)
  BlockCsrH PT;                       // transposed pattern (values built on the device)
  BigVec<int> tperm;                  // PT block d <- P block tperm[d] (2x2 transposed)
};

inline TransferPlan transfer_plan(const LevelPlan& C, const LevelPlan& F, const Refinement& R) {
  TransferPlan T;
  T.nrows = F.nb;
  T.ncols = C.nb;
  auto rows = averaging_blocks(C, F, R);
  T.avg.nrows = F.nb;
  T.avg.ncols = C.nb;
  T.avg.ptr.assign(F.nb + 1, 0);
  for (int rf = 0; rf < F.nb; ++rf) T.avg.ptr[rf + 1] = T.avg.ptr[rf] + rows[rf].n;
  T.avg.col.resize(T.avg.ptr[F.nb]);
  T.avg.val.resize(size_t(T.avg.ptr[F.nb]) * 4);
  parallel_for(F.nb, [&](int rf) {
    for (int q = 0; q < rows[rf].n; ++q) {
      const int d = T.avg.ptr[rf] + q;
      T.avg.col[d] = rows[rf].col[q];
      for (int t = 0; t < 4; ++t) T.avg.val[size_t(d) * 4 + t] = rows[rf].v[q][t];
    }
  });
  const TriMesh& fm = *F.mesh;
  T.nelem = int(R.children.size());
  T.nmed.assign(T.nelem, 0);
  T.med.assign(size_t(T.nelem) * 3, -1);
  for (int ff = 0; ff < fm.nf(); ++ff)
    if (R.fclass[ff] == kMedial && F.facet_block[ff] >= 0) {
      const int e = R.parent_elem[ff];
      T.med[size_t(e) * 3 + T.nmed[e]++] = F.facet_block[ff];
    }
  // correction columns from the pattern of A and of the averaging rows
  T.ncol.assign(T.nelem, 0);
  T.col.assign(size_t(T.nelem) * TransferPlan::kColMax, -1);
  ParArray<ColRow<kCorrCap>> rowcols(F.nb);  // per fine row: correction columns
  // the medial rows of different coarse elements are disjoint
  parallel_for(T.nelem, [&](int e) {
    ColRow<kCorrCap> cols;
    for (int i = 0; i < T.nmed[e]; ++i) {
      const int rb = T.med[size_t(e) * 3 + i];
      for (int sl = 0; sl < kSlots; ++sl) {
        const int jb = F.cols[size_t(rb) * kSlots + sl];
        if (jb < 0) continue;
        for (int q = 0; q < rows[jb].n; ++q) cols.add(rows[jb].col[q]);
      }
    }
    T.ncol[e] = cols.n;
    for (int j = 0; j < cols.n; ++j) T.col[size_t(e) * TransferPlan::kColMax + j] = cols.col[j];
    for (int i = 0; i < T.nmed[e]; ++i)
      for (int j = 0; j < cols.n; ++j) rowcols[T.med[size_t(e) * 3 + i]].add(cols.col[j]);
  });
  // final pattern: averaging columns + correction columns per fine row (sorted
  // merge of two small sorted lists; correction-only blocks start at zero)
  T.P.nrows = F.nb;
  T.P.ncols = C.nb;
  std::vector<int> cnt_row(F.nb);
  auto merge = [&](int rf, int* col, double* val) {
    const BlockRow<kAvgCap>& a = rows[rf];
    const ColRow<kCorrCap>& c = rowcols[rf];
    int i = 0, j = 0, n = 0;
    while (i < a.n || j < c.n) {
      const int ca = i < a.n ? a.col[i] : INT_MAX, cc = j < c.n ? c.col[j] : INT_MAX;
      const int cm = std::min(ca, cc);
      if (col) col[n] = cm;
      if (val)
        for (int t = 0; t < 4; ++t) val[size_t(n) * 4 + t] = ca == cm ? a.v[i][t] : 0.0;
      if (ca == cm) ++i;
      if (cc == cm) ++j;
      ++n;
    }
    return n;
  };
  parallel_for(F.nb, [&](int rf) { cnt_row[rf] = merge(rf, nullptr, nullptr); });
  T.P.ptr.assign(F.nb + 1, 0);
  for (int rf = 0; rf < F.nb; ++rf) T.P.ptr[rf + 1] = T.P.ptr[rf] + cnt_row[rf];
  T.P.col.resize(T.P.ptr[F.nb]);
  // P.val stays empty: the averaging values in P's pattern (the base the
  // correction is added to) are merged on the device (dev::prolong_base)
  parallel_for(F.nb, [&](int rf) { merge(rf, &T.P.col[T.P.ptr[rf]], nullptr); });
  T.pos.assign(size_t(T.nelem) * 3 * TransferPlan::kColMax, -1);
  parallel_for(T.nelem, [&](int e) {
    for (int i = 0; i < T.nmed[e]; ++i) {
      const int rb = T.med[size_t(e) * 3 + i];
      for (int j = 0; j < T.ncol[e]; ++j) {
        const int c = T.col[size_t(e) * TransferPlan::kColMax + j];
        for (int q = T.P.ptr[rb]; q < T.P.ptr[rb + 1]; ++q)
          if (T.P.col[q] == c) T.pos[(size_t(e) * 3 + i) * TransferPlan::kColMax + j] = q;
      }
    }
  });
  // transposed pattern and the block permutation
  T.PT.nrows = C.nb;
  T.PT.ncols = F.nb;
  std::vector<int> cnt(C.nb + 1, 0);
  for (int c : T.P.col) cnt[c + 1]++;
  for (int i = 0; i < C.nb; ++i) cnt[i + 1] += cnt[i];
  T.PT.ptr = cnt;
  T.PT.col.resize(T.P.col.size());  // every entry written by the scatter below
  T.tperm.resize(T.P.col.size());
  std::vector<int> at(cnt.begin(), cnt.end() - 1);
  for (int r = 0; r < F.nb; ++r)
    for (int q = T.P.ptr[r]; q < T.P.ptr[r + 1]; ++q) {
      const int d = at[T.P.col[q]]++;
      T.PT.col[d] = r;
      T.tperm[d] = q;
    }
  // PT.val stays empty: the device fills it from P (k_block_transpose_perm)
  return T;
}


}  // namespace host
}  // namespace hpmg
