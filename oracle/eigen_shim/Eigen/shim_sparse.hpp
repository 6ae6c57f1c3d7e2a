// TEST INFRASTRUCTURE ONLY (oracle/_ref): the Eigen 3 sparse subset the
// reference headers use (see shim_dense.hpp for the why). Always-compressed
// CSC / CSR storage with sorted inner indices; setFromTriplets sums
// duplicates in triplet order, products and sums follow Eigen's documented
// semantics (pattern union for +, explicit zeros kept until prune()).
#pragma once

#include "shim_dense.hpp"

namespace Eigen {

template <class S, class I = int>
class Triplet {
 public:
  Triplet() = default;
  Triplet(I r, I c, S v) : r_(r), c_(c), v_(v) {}
  I row() const { return r_; }
  I col() const { return c_; }
  S value() const { return v_; }

 private:
  I r_ = 0, c_ = 0;
  S v_ = 0;
};

template <class S, int Opt = ColMajor, class StorageIndex = int>
class SparseMatrix {
  static_assert(std::is_same<S, double>::value, "eigen shim: double only");

 public:
  using Scalar = double;
  static constexpr bool IsRowMajor = Opt == RowMajor;

  SparseMatrix() : outer_(1, 0) {}
  SparseMatrix(Index r, Index c) { resize(r, c); }
  template <int O2>
  SparseMatrix(const SparseMatrix<S, O2, StorageIndex>& o) {
    assign(o);
  }
  SparseMatrix(const SparseMatrix&) = default;
  SparseMatrix(SparseMatrix&&) = default;
  SparseMatrix& operator=(const SparseMatrix&) = default;
  SparseMatrix& operator=(SparseMatrix&&) = default;
  template <int O2>
  SparseMatrix& operator=(const SparseMatrix<S, O2, StorageIndex>& o) {
    SparseMatrix t;
    t.assign(o);
    *this = std::move(t);
    return *this;
  }

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index outerSize() const { return IsRowMajor ? rows_ : cols_; }
  Index innerSize() const { return IsRowMajor ? cols_ : rows_; }
  Index nonZeros() const { return Index(val_.size()); }
  void resize(Index r, Index c) {
    rows_ = r;
    cols_ = c;
    outer_.assign(std::size_t(outerSize() + 1), 0);
    inner_.clear();
    val_.clear();
  }
  void makeCompressed() {}
  bool isCompressed() const { return true; }
  void reserve(Index) {}
  void setZero() { resize(rows_, cols_); }

  template <class It>
  void setFromTriplets(It begin, It end) {
    // bucket by outer index keeping triplet order, then sort each outer
    // vector stably by inner index and sum duplicates in triplet order
    const Index no = outerSize();
    std::vector<Index> count(std::size_t(no + 1), 0);
    std::size_t nt = 0;
    for (It it = begin; it != end; ++it, ++nt) ++count[std::size_t(outer_of(*it) + 1)];
    for (Index o = 0; o < no; ++o) count[std::size_t(o + 1)] += count[std::size_t(o)];
    std::vector<std::pair<Index, double>> e(nt);
    std::vector<Index> pos(count.begin(), count.end() - 1);
    for (It it = begin; it != end; ++it)
      e[std::size_t(pos[std::size_t(outer_of(*it))]++)] = {inner_of(*it), double(it->value())};
    outer_.assign(std::size_t(no + 1), 0);
    inner_.clear();
    val_.clear();
    inner_.reserve(nt);
    val_.reserve(nt);
    for (Index o = 0; o < no; ++o) {
      auto b = e.begin() + count[std::size_t(o)], en = e.begin() + count[std::size_t(o + 1)];
      std::stable_sort(b, en, [](const auto& x, const auto& y) { return x.first < y.first; });
      for (auto p = b; p != en; ++p) {
        if (!inner_.empty() && Index(inner_.size()) > outer_[std::size_t(o)] &&
            inner_.back() == StorageIndex(p->first))
          val_.back() += p->second;
        else {
          inner_.push_back(StorageIndex(p->first));
          val_.push_back(p->second);
        }
      }
      outer_[std::size_t(o + 1)] = Index(inner_.size());
    }
  }

  /// Removes entries with |v| <= |reference| * epsilon (reference 0: exact
  /// zeros only).
  void prune(double reference, double epsilon = 1e-12) {
    std::size_t w = 0;
    std::vector<Index> no(outer_.size(), 0);
    for (Index o = 0; o < outerSize(); ++o) {
      for (Index p = outer_[std::size_t(o)]; p < outer_[std::size_t(o + 1)]; ++p)
        if (std::abs(val_[std::size_t(p)]) > std::abs(reference) * epsilon) {
          inner_[w] = inner_[std::size_t(p)];
          val_[w] = val_[std::size_t(p)];
          ++w;
        }
      no[std::size_t(o + 1)] = Index(w);
    }
    outer_ = no;
    inner_.resize(w);
    val_.resize(w);
  }

  double coeff(Index r, Index c) const {
    const Index o = IsRowMajor ? r : c, in = IsRowMajor ? c : r;
    auto b = inner_.begin() + outer_[std::size_t(o)], e = inner_.begin() + outer_[std::size_t(o + 1)];
    auto it = std::lower_bound(b, e, StorageIndex(in));
    if (it == e || *it != StorageIndex(in)) return 0.0;
    return val_[std::size_t(it - inner_.begin())];
  }

  class InnerIterator {
   public:
    InnerIterator(const SparseMatrix& m, Index outer)
        : m_(&m), o_(outer), p_(m.outer_[std::size_t(outer)]), e_(m.outer_[std::size_t(outer + 1)]) {}
    explicit operator bool() const { return p_ < e_; }
    InnerIterator& operator++() {
      ++p_;
      return *this;
    }
    double value() const { return m_->val_[std::size_t(p_)]; }
    Index index() const { return m_->inner_[std::size_t(p_)]; }
    Index outer() const { return o_; }
    Index row() const { return IsRowMajor ? o_ : index(); }
    Index col() const { return IsRowMajor ? index() : o_; }

   private:
    const SparseMatrix* m_;
    Index o_, p_, e_;
  };

  /// The transpose shares the arrays, reinterpreted in the other order.
  SparseMatrix<S, 1 - Opt, StorageIndex> transpose() const {
    SparseMatrix<S, 1 - Opt, StorageIndex> t;
    t.rows_ = cols_;
    t.cols_ = rows_;
    t.outer_ = outer_;
    t.inner_ = inner_;
    t.val_ = val_;
    return t;
  }

  double* valuePtr() { return val_.data(); }
  const double* valuePtr() const { return val_.data(); }
  const StorageIndex* innerIndexPtr() const { return inner_.data(); }
  const Index* outerIndexPtr() const { return outer_.data(); }

  SparseMatrix& operator*=(double a) {
    for (double& v : val_) v *= a;
    return *this;
  }

  // data shared by all instantiations
  Index rows_ = 0, cols_ = 0;
  std::vector<Index> outer_;
  std::vector<StorageIndex> inner_;
  std::vector<double> val_;

 private:
  template <class T>
  Index outer_of(const T& t) const {
    return IsRowMajor ? Index(t.row()) : Index(t.col());
  }
  template <class T>
  Index inner_of(const T& t) const {
    return IsRowMajor ? Index(t.col()) : Index(t.row());
  }
  template <int O2>
  void assign(const SparseMatrix<S, O2, StorageIndex>& o) {
    rows_ = o.rows_;
    cols_ = o.cols_;
    if (O2 == Opt) {
      outer_ = o.outer_;
      inner_ = o.inner_;
      val_ = o.val_;
      return;
    }
    // storage-order change: counting transpose (inner indices stay sorted)
    const Index no = outerSize();
    outer_.assign(std::size_t(no + 1), 0);
    for (auto i : o.inner_) ++outer_[std::size_t(i + 1)];
    for (Index k = 0; k < no; ++k) outer_[std::size_t(k + 1)] += outer_[std::size_t(k)];
    inner_.assign(o.inner_.size(), 0);
    val_.assign(o.val_.size(), 0.0);
    std::vector<Index> pos(outer_.begin(), outer_.end() - 1);
    for (Index oo = 0; oo < o.outerSize(); ++oo)
      for (Index p = o.outer_[std::size_t(oo)]; p < o.outer_[std::size_t(oo + 1)]; ++p) {
        const Index q = pos[std::size_t(o.inner_[std::size_t(p)])]++;
        inner_[std::size_t(q)] = StorageIndex(oo);
        val_[std::size_t(q)] = o.val_[std::size_t(p)];
      }
  }
};

// dense conversion: Mat(sparse)
template <class S, int O, class I>
MatrixXd to_dense(const SparseMatrix<S, O, I>& a) {
  MatrixXd m = MatrixXd::Zero(a.rows(), a.cols());
  for (Index o = 0; o < a.outerSize(); ++o)
    for (typename SparseMatrix<S, O, I>::InnerIterator it(a, o); it; ++it) m(it.row(), it.col()) += it.value();
  return m;
}

// sparse * dense vector/matrix: column-major scatter (y += x_j * A(:,j)),
// row-major gather (y_i = sum_k A(i,k) x_k)
template <class S, int O, class I, class B, std::enable_if_t<is_dense_v<B>, int> = 0>
auto operator*(const SparseMatrix<S, O, I>& a, const B& b) {
  if (a.cols() != b.rows()) throw std::logic_error("eigen shim: spmv size mismatch");
  Matrix<double, Dynamic, internal::traits<std::decay_t<B>>::cols> y =
      Matrix<double, Dynamic, internal::traits<std::decay_t<B>>::cols>::Zero(a.rows(), b.cols());
  for (Index c = 0; c < b.cols(); ++c) {
    if (O == ColMajor) {
      for (Index j = 0; j < a.outerSize(); ++j) {
        const double xj = b(j, c);
        for (Index p = a.outer_[std::size_t(j)]; p < a.outer_[std::size_t(j + 1)]; ++p)
          y(a.inner_[std::size_t(p)], c) += a.val_[std::size_t(p)] * xj;
      }
    } else {
      for (Index i = 0; i < a.outerSize(); ++i) {
        double s = 0;
        for (Index p = a.outer_[std::size_t(i)]; p < a.outer_[std::size_t(i + 1)]; ++p)
          s += a.val_[std::size_t(p)] * b(a.inner_[std::size_t(p)], c);
        y(i, c) = s;
      }
    }
  }
  return y;
}

// sparse * sparse: column j of the product accumulates B(k,j) A(:,k) over
// ascending k (Eigen's conservative product), result column-major sorted.
template <class S, int O1, int O2, class I>
SparseMatrix<S, ColMajor, I> operator*(const SparseMatrix<S, O1, I>& a0, const SparseMatrix<S, O2, I>& b0) {
  const SparseMatrix<S, ColMajor, I> a(a0), b(b0);
  if (a.cols() != b.rows()) throw std::logic_error("eigen shim: spgemm size mismatch");
  SparseMatrix<S, ColMajor, I> r(a.rows(), b.cols());
  std::vector<double> acc(std::size_t(a.rows()), 0.0);
  std::vector<char> mark(std::size_t(a.rows()), 0);
  std::vector<Index> rows;
  for (Index j = 0; j < b.cols(); ++j) {
    rows.clear();
    for (Index pb = b.outer_[std::size_t(j)]; pb < b.outer_[std::size_t(j + 1)]; ++pb) {
      const Index k = b.inner_[std::size_t(pb)];
      const double bkj = b.val_[std::size_t(pb)];
      for (Index pa = a.outer_[std::size_t(k)]; pa < a.outer_[std::size_t(k + 1)]; ++pa) {
        const Index i = a.inner_[std::size_t(pa)];
        if (!mark[std::size_t(i)]) {
          mark[std::size_t(i)] = 1;
          acc[std::size_t(i)] = a.val_[std::size_t(pa)] * bkj;
          rows.push_back(i);
        } else {
          acc[std::size_t(i)] += a.val_[std::size_t(pa)] * bkj;
        }
      }
    }
    std::sort(rows.begin(), rows.end());
    for (Index i : rows) {
      r.inner_.push_back(I(i));
      r.val_.push_back(acc[std::size_t(i)]);
      mark[std::size_t(i)] = 0;
    }
    r.outer_[std::size_t(j + 1)] = Index(r.inner_.size());
  }
  return r;
}

template <class S, int O, class I>
SparseMatrix<S, O, I> operator*(double s, const SparseMatrix<S, O, I>& a) {
  SparseMatrix<S, O, I> r(a);
  for (double& v : r.val_) v = s * v;
  return r;
}
template <class S, int O, class I>
SparseMatrix<S, O, I> operator*(const SparseMatrix<S, O, I>& a, double s) {
  SparseMatrix<S, O, I> r(a);
  for (double& v : r.val_) v = v * s;
  return r;
}

// sum over the union of the two patterns
template <class S, int O, class I>
SparseMatrix<S, O, I> sparse_combine(const SparseMatrix<S, O, I>& a, const SparseMatrix<S, O, I>& b, double sb) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) throw std::logic_error("eigen shim: sparse sum size");
  SparseMatrix<S, O, I> r(a.rows(), a.cols());
  for (Index o = 0; o < a.outerSize(); ++o) {
    Index pa = a.outer_[std::size_t(o)], ea = a.outer_[std::size_t(o + 1)];
    Index pb = b.outer_[std::size_t(o)], eb = b.outer_[std::size_t(o + 1)];
    while (pa < ea || pb < eb) {
      const Index ia = pa < ea ? Index(a.inner_[std::size_t(pa)]) : std::numeric_limits<Index>::max();
      const Index ib = pb < eb ? Index(b.inner_[std::size_t(pb)]) : std::numeric_limits<Index>::max();
      if (ia == ib) {
        r.inner_.push_back(I(ia));
        r.val_.push_back(a.val_[std::size_t(pa++)] + sb * b.val_[std::size_t(pb++)]);
      } else if (ia < ib) {
        r.inner_.push_back(I(ia));
        r.val_.push_back(a.val_[std::size_t(pa++)]);
      } else {
        r.inner_.push_back(I(ib));
        r.val_.push_back(sb * b.val_[std::size_t(pb++)]);
      }
    }
    r.outer_[std::size_t(o + 1)] = Index(r.inner_.size());
  }
  return r;
}
template <class S, int O, class I>
SparseMatrix<S, O, I> operator+(const SparseMatrix<S, O, I>& a, const SparseMatrix<S, O, I>& b) {
  return sparse_combine(a, b, 1.0);
}
template <class S, int O, class I>
SparseMatrix<S, O, I> operator-(const SparseMatrix<S, O, I>& a, const SparseMatrix<S, O, I>& b) {
  return sparse_combine(a, b, -1.0);
}

}  // namespace Eigen
