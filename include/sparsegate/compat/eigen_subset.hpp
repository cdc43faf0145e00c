// sparsegate-b200 — an eagerly evaluated subset of the Eigen 3.3 dense API, used
// by include/sparsegate/common.hpp ONLY when the real <Eigen/Dense> is not on the
// include path (this image has no Eigen). It is the container the
// reference's Mat / Vec are (common.hpp:15-18) with the members the reference's
// headers, callers and tests use:
//   * the reference's own headers compile unmodified against it into oracle/_ref/
//     ({common,types,ffn_exec,synthetic,calibration}.hpp; oracle/Makefile), and
//   * the reference's own tests compile unmodified against this repo's drop-in
//     headers (tests/cpp/Makefile: proj/tests/ffn_exec_tests.cpp).
// A user with Eigen installed gets the real library instead.
//
// Semantics kept from Eigen: storage order (the reference's Mat is RowMajor,
// common.hpp:16; VectorXd is a contiguous column), comma initialisation row by
// row, coefficient-wise Array arithmetic vs. matrix products, colwise()
// reductions / broadcasts, isZero with the double dummy precision 1e-12.
// Products and reductions are plain ascending loops: no Eigen arithmetic
// decides a bit of the executor output (every executor dot product goes
// through det_dot / det_sum, ffn_exec.hpp:96-98).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
constexpr int RowMajor = 1;
constexpr int ColMajor = 0;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

template <typename S, int R, int C, int O, bool IsArray>
class Dense;

template <typename S, int R, int C, int O = ColMajor, int MR = R, int MC = C>
using Matrix = Dense<S, R, C, O, false>;
template <typename S, int R, int C, int O = ColMajor, int MR = R, int MC = C>
using Array = Dense<S, R, C, O, true>;

using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXi = Matrix<int, Dynamic, 1>;
using ArrayXd = Array<double, Dynamic, 1>;
using ArrayXXd = Array<double, Dynamic, Dynamic>;

template <typename D>
class CommaInit;
template <typename D>
class Vectorwise;

template <typename S, int R, int C, int O, bool IsArray>
class Dense {
  public:
    using Scalar = S;
    static constexpr bool kRowMajor = (O & RowMajor) != 0 || (R == 1 && C != 1);

    Dense() : rows_(R > 0 ? R : 0), cols_(C > 0 ? C : 0), v_(static_cast<std::size_t>(rows_ * cols_)) {}
    // vector constructor (one of the dimensions fixed to 1), or (rows, cols)
    explicit Dense(Index n) : rows_(C == 1 ? n : 1), cols_(C == 1 ? 1 : n), v_(static_cast<std::size_t>(n)) {}
    Dense(Index r, Index c) : rows_(r), cols_(c), v_(static_cast<std::size_t>(r * c)) {}
    // conversion between storage orders, Matrix <-> Array, vector shapes
    template <int R2, int C2, int O2, bool A2>
    Dense(const Dense<S, R2, C2, O2, A2>& o) : rows_(o.rows()), cols_(o.cols()), v_(o.size()) {
        if (C == 1 && o.cols() != 1 && o.rows() == 1) {  // row vector -> column vector
            rows_ = o.cols();
            cols_ = 1;
        }
        for (Index i = 0; i < rows_; ++i)
            for (Index j = 0; j < cols_; ++j)
                (*this)(i, j) = (C == 1 && o.cols() != 1) ? o(0, i) : o(i, j);
    }

    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index size() const { return rows_ * cols_; }
    S* data() { return v_.data(); }
    const S* data() const { return v_.data(); }

    void resize(Index n) {
        rows_ = C == 1 ? n : 1;
        cols_ = C == 1 ? 1 : n;
        v_.assign(static_cast<std::size_t>(n), S(0));
    }
    void resize(Index r, Index c) {
        rows_ = r;
        cols_ = c;
        v_.assign(static_cast<std::size_t>(r * c), S(0));
    }

    S& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
    const S& operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }
    S& operator[](Index i) { return v_[static_cast<std::size_t>(i)]; }
    const S& operator[](Index i) const { return v_[static_cast<std::size_t>(i)]; }
    S& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(off(i, j))]; }
    const S& operator()(Index i, Index j) const { return v_[static_cast<std::size_t>(off(i, j))]; }
    S coeff(Index i, Index j) const { return (*this)(i, j); }

    // ---- initialisation ----
    Dense& setConstant(S s) {
        std::fill(v_.begin(), v_.end(), s);
        return *this;
    }
    Dense& setZero() { return setConstant(S(0)); }
    Dense& setOnes() { return setConstant(S(1)); }
    void fill(S s) { setConstant(s); }
    static Dense Constant(Index r, Index c, S s) { return Dense(r, c).setConstant(s); }
    static Dense Constant(Index n, S s) { return Dense(n).setConstant(s); }
    static Dense Zero(Index r, Index c) { return Constant(r, c, S(0)); }
    static Dense Zero(Index n) { return Constant(n, S(0)); }
    static Dense Ones(Index r, Index c) { return Constant(r, c, S(1)); }
    static Dense Ones(Index n) { return Constant(n, S(1)); }
    static Dense Identity(Index r, Index c) {
        Dense m = Zero(r, c);
        for (Index i = 0; i < r && i < c; ++i) m(i, i) = S(1);
        return m;
    }
    static Dense Identity(Index n) { return Identity(n, n); }
    CommaInit<Dense> operator<<(S s);

    // ---- element-wise / reductions ----
    bool allFinite() const {
        for (const S& s : v_)
            if (!std::isfinite(static_cast<double>(s))) return false;
        return true;
    }
    bool hasNaN() const {
        for (const S& s : v_)
            if (std::isnan(static_cast<double>(s))) return true;
        return false;
    }
    bool isZero(double prec = 1e-12) const {
        for (const S& s : v_)
            if (!(std::abs(static_cast<double>(s)) <= prec)) return false;
        return true;
    }
    S sum() const {
        S a = S(0);
        for (Index i = 0; i < rows_; ++i)
            for (Index j = 0; j < cols_; ++j) a += (*this)(i, j);
        return a;
    }
    S mean() const { return sum() / static_cast<S>(size()); }
    S trace() const {
        S a = S(0);
        for (Index i = 0; i < rows_ && i < cols_; ++i) a += (*this)(i, i);
        return a;
    }
    S squaredNorm() const {
        S a = S(0);
        for (Index i = 0; i < rows_; ++i)
            for (Index j = 0; j < cols_; ++j) a += (*this)(i, j) * (*this)(i, j);
        return a;
    }
    S norm() const { return std::sqrt(squaredNorm()); }
    S minCoeff() const { return *std::min_element(v_.begin(), v_.end()); }
    S maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }
    template <int R2, int C2, int O2, bool A2>
    S dot(const Dense<S, R2, C2, O2, A2>& o) const {
        need(size() == o.size(), "dot: size mismatch");
        S a = S(0);
        for (Index i = 0; i < size(); ++i) a += lin(i) * o.lin(i);
        return a;
    }
    bool any() const {
        for (const S& s : v_)
            if (s) return true;
        return false;
    }
    bool all() const {
        for (const S& s : v_)
            if (!s) return false;
        return true;
    }
    Index count() const {
        Index n = 0;
        for (const S& s : v_) n += s ? 1 : 0;
        return n;
    }

    template <typename F>
    Dense unary(F f) const {
        Dense out(*this);
        for (S& s : out.v_) s = f(s);
        return out;
    }
    template <typename F, int R2, int C2, int O2, bool A2>
    Dense binary(const Dense<S, R2, C2, O2, A2>& o, F f) const {
        need(rows_ == o.rows() && cols_ == o.cols(), "coefficient-wise op: shape mismatch");
        Dense out(rows_, cols_);
        for (Index i = 0; i < rows_; ++i)
            for (Index j = 0; j < cols_; ++j) out(i, j) = f((*this)(i, j), o(i, j));
        return out;
    }
    Dense cwiseMax(S s) const { return unary([s](S a) { return a > s ? a : s; }); }
    Dense cwiseMin(S s) const { return unary([s](S a) { return a < s ? a : s; }); }
    Dense cwiseAbs() const { return unary([](S a) { return std::abs(a); }); }
    Dense cwiseSqrt() const { return unary([](S a) { return std::sqrt(a); }); }
    Dense cwiseAbs2() const { return unary([](S a) { return a * a; }); }
    template <int R2, int C2, int O2, bool A2>
    Dense cwiseMax(const Dense<S, R2, C2, O2, A2>& o) const {
        return binary(o, [](S a, S b) { return a > b ? a : b; });
    }
    template <int R2, int C2, int O2, bool A2>
    Dense cwiseMin(const Dense<S, R2, C2, O2, A2>& o) const {
        return binary(o, [](S a, S b) { return a < b ? a : b; });
    }
    template <int R2, int C2, int O2, bool A2>
    Dense cwiseProduct(const Dense<S, R2, C2, O2, A2>& o) const {
        return binary(o, [](S a, S b) { return a * b; });
    }
    template <int R2, int C2, int O2, bool A2>
    Dense cwiseQuotient(const Dense<S, R2, C2, O2, A2>& o) const {
        return binary(o, [](S a, S b) { return a / b; });
    }
    // Array functions
    Dense square() const { return cwiseAbs2(); }
    Dense abs() const { return cwiseAbs(); }
    Dense sqrt() const { return cwiseSqrt(); }
    Dense exp() const { return unary([](S a) { return std::exp(a); }); }
    Dense log() const { return unary([](S a) { return std::log(a); }); }

    // ---- views (copies) ----
    Dense eval() const { return *this; }
    Dense<S, C, R, (R == 1 || C == 1) ? O : (O ^ RowMajor), IsArray> transpose() const {
        Dense<S, C, R, (R == 1 || C == 1) ? O : (O ^ RowMajor), IsArray> t(cols_, rows_);
        for (Index i = 0; i < rows_; ++i)
            for (Index j = 0; j < cols_; ++j) t(j, i) = (*this)(i, j);
        return t;
    }
    Dense<S, R, C, O, true> array() const { return Dense<S, R, C, O, true>(*this); }
    Dense<S, R, C, O, false> matrix() const { return Dense<S, R, C, O, false>(*this); }
    Vectorwise<Dense> colwise() const { return Vectorwise<Dense>(*this, true); }
    Vectorwise<Dense> rowwise() const { return Vectorwise<Dense>(*this, false); }
    Dense<S, Dynamic, Dynamic, O, IsArray> block(Index i0, Index j0, Index r, Index c) const {
        need(i0 >= 0 && j0 >= 0 && i0 + r <= rows_ && j0 + c <= cols_, "block out of range");
        Dense<S, Dynamic, Dynamic, O, IsArray> b(r, c);
        for (Index i = 0; i < r; ++i)
            for (Index j = 0; j < c; ++j) b(i, j) = (*this)(i0 + i, j0 + j);
        return b;
    }
    Dense<S, Dynamic, 1, ColMajor, IsArray> col(Index j) const {
        Dense<S, Dynamic, 1, ColMajor, IsArray> v(rows_);
        for (Index i = 0; i < rows_; ++i) v(i) = (*this)(i, j);
        return v;
    }
    Dense<S, 1, Dynamic, RowMajor, IsArray> row(Index i) const {
        Dense<S, 1, Dynamic, RowMajor, IsArray> v(1, cols_);
        for (Index j = 0; j < cols_; ++j) v(0, j) = (*this)(i, j);
        return v;
    }
    Dense<S, Dynamic, Dynamic, O, IsArray> leftCols(Index n) const { return block(0, 0, rows_, n); }
    Dense<S, Dynamic, Dynamic, O, IsArray> rightCols(Index n) const { return block(0, cols_ - n, rows_, n); }
    Dense<S, Dynamic, Dynamic, O, IsArray> topRows(Index n) const { return block(0, 0, n, cols_); }
    Dense<S, Dynamic, Dynamic, O, IsArray> bottomRows(Index n) const { return block(rows_ - n, 0, n, cols_); }
    Dense segment(Index i, Index n) const {
        need(i >= 0 && i + n <= size(), "segment out of range");
        Dense v(n);
        for (Index k = 0; k < n; ++k) v(k) = lin(i + k);
        return v;
    }
    Dense head(Index n) const { return segment(0, n); }
    Dense tail(Index n) const { return segment(size() - n, n); }
    Dense<S, Dynamic, Dynamic, ColMajor, false> asDiagonal() const {
        Dense<S, Dynamic, Dynamic, ColMajor, false> m = Dense<S, Dynamic, Dynamic, ColMajor, false>::Zero(size(), size());
        for (Index i = 0; i < size(); ++i) m(i, i) = lin(i);
        return m;
    }
    template <typename T>
    Dense<T, R, C, O, IsArray> cast() const {
        Dense<T, R, C, O, IsArray> out(rows_, cols_);
        for (Index i = 0; i < rows_; ++i)
            for (Index j = 0; j < cols_; ++j) out(i, j) = static_cast<T>((*this)(i, j));
        return out;
    }

    // ---- arithmetic ----
    template <int R2, int C2, int O2, bool A2>
    Dense operator+(const Dense<S, R2, C2, O2, A2>& o) const {
        return binary(o, [](S a, S b) { return a + b; });
    }
    template <int R2, int C2, int O2, bool A2>
    Dense operator-(const Dense<S, R2, C2, O2, A2>& o) const {
        return binary(o, [](S a, S b) { return a - b; });
    }
    Dense operator-() const { return unary([](S a) { return -a; }); }
    Dense operator*(S s) const { return unary([s](S a) { return a * s; }); }
    Dense operator/(S s) const { return unary([s](S a) { return a / s; }); }
    friend Dense operator*(S s, const Dense& m) { return m * s; }
    Dense operator+(S s) const { return unary([s](S a) { return a + s; }); }
    Dense operator-(S s) const { return unary([s](S a) { return a - s; }); }
    template <int R2, int C2, int O2, bool A2>
    Dense& operator+=(const Dense<S, R2, C2, O2, A2>& o) {
        return *this = *this + o;
    }
    template <int R2, int C2, int O2, bool A2>
    Dense& operator-=(const Dense<S, R2, C2, O2, A2>& o) {
        return *this = *this - o;
    }
    Dense& operator*=(S s) { return *this = *this * s; }
    Dense& operator/=(S s) { return *this = *this / s; }
    // Matrix: product; Array: coefficient-wise
    template <int R2, int C2, int O2, bool A2>
    Dense<S, R, C2, O, IsArray> operator*(const Dense<S, R2, C2, O2, A2>& b) const {
        if constexpr (IsArray) {
            return binary(b, [](S x, S y) { return x * y; });
        } else {
            need(cols_ == b.rows(), "product shape mismatch");
            Dense<S, R, C2, O, IsArray> out(rows_, b.cols());
            for (Index i = 0; i < rows_; ++i)
                for (Index j = 0; j < b.cols(); ++j) {
                    S a = S(0);
                    for (Index k = 0; k < cols_; ++k) a += (*this)(i, k) * b(k, j);
                    out(i, j) = a;
                }
            return out;
        }
    }
    template <int R2, int C2, int O2, bool A2>
    Dense operator/(const Dense<S, R2, C2, O2, A2>& o) const {
        return binary(o, [](S a, S b) { return a / b; });
    }
    // Array comparisons with a scalar -> boolean array
    Dense<int, R, C, O, true> operator<(S s) const { return cmp([s](S a) { return a < s; }); }
    Dense<int, R, C, O, true> operator<=(S s) const { return cmp([s](S a) { return a <= s; }); }
    Dense<int, R, C, O, true> operator>(S s) const { return cmp([s](S a) { return a > s; }); }
    Dense<int, R, C, O, true> operator>=(S s) const { return cmp([s](S a) { return a >= s; }); }
    template <int R2, int C2, int O2, bool A2>
    bool operator==(const Dense<S, R2, C2, O2, A2>& o) const {
        if (rows_ != o.rows() || cols_ != o.cols()) return false;
        for (Index i = 0; i < rows_; ++i)
            for (Index j = 0; j < cols_; ++j)
                if ((*this)(i, j) != o(i, j)) return false;
        return true;
    }
    template <int R2, int C2, int O2, bool A2>
    bool operator!=(const Dense<S, R2, C2, O2, A2>& o) const {
        return !(*this == o);
    }

    // linear (storage-order independent for vectors) access
    S lin(Index k) const { return (rows_ == 1 || cols_ == 1) ? v_[static_cast<std::size_t>(k)] : (*this)(k / cols_, k % cols_); }
    static void need(bool ok, const char* what) {
        if (!ok) throw std::invalid_argument(std::string("eigen shim: ") + what);
    }

  private:
    template <typename F>
    Dense<int, R, C, O, true> cmp(F f) const {
        Dense<int, R, C, O, true> out(rows_, cols_);
        for (Index i = 0; i < rows_; ++i)
            for (Index j = 0; j < cols_; ++j) out(i, j) = f((*this)(i, j));
        return out;
    }
    Index off(Index i, Index j) const { return kRowMajor ? i * cols_ + j : j * rows_ + i; }

    Index rows_ = 0;
    Index cols_ = 0;
    std::vector<S> v_;
};

// `m << a, b, c, ...` fills row by row (Eigen's comma initializer order).
template <typename D>
class CommaInit {
  public:
    CommaInit(D& m, typename D::Scalar s) : m_(m) { put(s); }
    CommaInit& operator,(typename D::Scalar s) {
        put(s);
        return *this;
    }

  private:
    void put(typename D::Scalar s) {
        D::need(k_ < m_.size(), "too many coefficients in comma initializer");
        m_(k_ / m_.cols(), k_ % m_.cols()) = s;
        ++k_;
    }
    D& m_;
    Index k_ = 0;
};
template <typename S, int R, int C, int O, bool A>
CommaInit<Dense<S, R, C, O, A>> Dense<S, R, C, O, A>::operator<<(S s) {
    return CommaInit<Dense>(*this, s);
}

// colwise() / rowwise(): reductions per column (row) and broadcasts of a vector
// over the columns (rows).
template <typename D>
class Vectorwise {
  public:
    using S = typename D::Scalar;
    Vectorwise(const D& m, bool cols) : m_(m), cols_(cols) {}
    template <typename F>
    Dense<S, Dynamic, Dynamic, RowMajor, false> reduce(F f) const {
        const Index n = cols_ ? m_.cols() : m_.rows(), len = cols_ ? m_.rows() : m_.cols();
        Dense<S, Dynamic, Dynamic, RowMajor, false> out(cols_ ? 1 : n, cols_ ? n : 1);
        for (Index k = 0; k < n; ++k) {
            std::vector<S> v(static_cast<std::size_t>(len));
            for (Index i = 0; i < len; ++i) v[static_cast<std::size_t>(i)] = cols_ ? m_(i, k) : m_(k, i);
            out(cols_ ? 0 : k, cols_ ? k : 0) = f(v);
        }
        return out;
    }
    Dense<S, Dynamic, Dynamic, RowMajor, false> squaredNorm() const {
        return reduce([](const std::vector<S>& v) {
            S a = S(0);
            for (S x : v) a += x * x;
            return a;
        });
    }
    Dense<S, Dynamic, Dynamic, RowMajor, false> norm() const {
        return reduce([](const std::vector<S>& v) {
            S a = S(0);
            for (S x : v) a += x * x;
            return std::sqrt(a);
        });
    }
    Dense<S, Dynamic, Dynamic, RowMajor, false> sum() const {
        return reduce([](const std::vector<S>& v) {
            S a = S(0);
            for (S x : v) a += x;
            return a;
        });
    }
    Dense<S, Dynamic, Dynamic, RowMajor, false> maxCoeff() const {
        return reduce([](const std::vector<S>& v) { return *std::max_element(v.begin(), v.end()); });
    }
    Dense<S, Dynamic, Dynamic, RowMajor, false> minCoeff() const {
        return reduce([](const std::vector<S>& v) { return *std::min_element(v.begin(), v.end()); });
    }
    // broadcast: colwise() op column vector (length rows), rowwise() op row vector
    template <int R2, int C2, int O2, bool A2>
    D operator*(const Dense<S, R2, C2, O2, A2>& v) const {
        return apply(v, [](S a, S b) { return a * b; });
    }
    template <int R2, int C2, int O2, bool A2>
    D operator+(const Dense<S, R2, C2, O2, A2>& v) const {
        return apply(v, [](S a, S b) { return a + b; });
    }
    template <int R2, int C2, int O2, bool A2>
    D operator-(const Dense<S, R2, C2, O2, A2>& v) const {
        return apply(v, [](S a, S b) { return a - b; });
    }

  private:
    template <typename V, typename F>
    D apply(const V& v, F f) const {
        D out(m_);
        D::need(v.size() == (cols_ ? m_.rows() : m_.cols()), "broadcast length mismatch");
        for (Index i = 0; i < m_.rows(); ++i)
            for (Index j = 0; j < m_.cols(); ++j) out(i, j) = f(m_(i, j), v.lin(cols_ ? i : j));
        return out;
    }
    D m_;
    bool cols_;
};

}  // namespace Eigen
