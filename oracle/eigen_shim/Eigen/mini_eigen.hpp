// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// A small stand-in for the Eigen API subset the reference headers use
// (/root/reference/proj/include/specmesh/{core,mesh,partition,spectral,pipeline}.hpp),
// so that the reference's OWN unmodified sources compile and run in this
// container (Eigen is a third-party dependency of the reference that is absent
// here: no version pinned, CMakeLists.txt:5 expects it under proj/vendor/).
//
// What this pins: every line of the reference's own code -- control flow,
// thresholds, tie rules, RNG draws, operation order of the shift, the DOI
// controller, segmentation, stitching.  What it does not pin: the rounding of
// Eigen's inner numerical kernels, which are restated here from their published
// algorithms (call sites in the reference: spectral.hpp:66, :96, :125-129,
// :155-156, :168, :174, :307):
//   HouseholderQR            unblocked Householder QR, Eigen's reflector convention
//                            (beta = -sign(x0)|x|, tau = (beta-x0)/beta, v = [1; x_tail/(x0-beta)])
//   SimplicialLDLT           envelope (skyline) L D L^T without pivoting under a reverse
//                            Cuthill-McKee ordering (Eigen: AMD ordering; same factorisation
//                            up to the permutation, i.e. up to rounding)
//   SelfAdjointEigenSolver   Householder tridiagonalisation + implicit-shift QL
//   JacobiSVD                one-sided (Hestenes) Jacobi, singular values only
//   dense products           plain loops, k-sequential accumulation
// Everything is evaluated eagerly (no expression templates); block accessors on
// non-const matrices return writable views, on const matrices copies.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum NoChange_t { NoChange };

template <typename T>
class Mat;
template <typename M>
class BlockRef;
template <typename M>
class JacobiSVD;
template <typename T>
class SparseMatrix;

namespace shim_detail {
inline void fail(const char* what) { throw std::logic_error(std::string("eigen shim: ") + what); }
}  // namespace shim_detail

// Column-major dense matrix with run-time shape.  All arithmetic returns Mat.
template <typename T>
class Mat {
protected:
    Index r_ = 0, c_ = 0;
    std::vector<T> d_;

public:
    using Scalar = T;
    Mat() = default;
    Mat(Index r, Index c) : r_(r), c_(c), d_(static_cast<std::size_t>(r * c), T()) {}

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    T* data() { return d_.data(); }
    const T* data() const { return d_.data(); }

    T& operator()(Index i, Index j) { return d_[static_cast<std::size_t>(j * r_ + i)]; }
    const T& operator()(Index i, Index j) const { return d_[static_cast<std::size_t>(j * r_ + i)]; }
    T& operator()(Index i) { return d_[static_cast<std::size_t>(i)]; }
    const T& operator()(Index i) const { return d_[static_cast<std::size_t>(i)]; }
    T& operator[](Index i) { return d_[static_cast<std::size_t>(i)]; }
    const T& operator[](Index i) const { return d_[static_cast<std::size_t>(i)]; }

    void resize(Index r, Index c) {
        if (r == r_ && c == c_) return;
        r_ = r;
        c_ = c;
        d_.assign(static_cast<std::size_t>(r * c), T());
    }
    // keeps the leading columns (column-major storage)
    void conservativeResize(NoChange_t, Index nc) {
        d_.resize(static_cast<std::size_t>(r_ * nc), T());
        c_ = nc;
    }
    void setZero() { std::fill(d_.begin(), d_.end(), T()); }
    void setConstant(T v) { std::fill(d_.begin(), d_.end(), v); }
    const Mat& eval() const { return *this; }

    // ---- blocks: views on non-const, copies on const
    BlockRef<Mat> row(Index i) { return BlockRef<Mat>(*this, i, 0, 1, c_); }
    BlockRef<Mat> col(Index j) { return BlockRef<Mat>(*this, 0, j, r_, 1); }
    BlockRef<Mat> leftCols(Index n) { return BlockRef<Mat>(*this, 0, 0, r_, n); }
    BlockRef<Mat> topRows(Index n) { return BlockRef<Mat>(*this, 0, 0, n, c_); }
    Mat block_copy(Index r0, Index c0, Index nr, Index nc) const {
        Mat out(nr, nc);
        for (Index j = 0; j < nc; ++j)
            for (Index i = 0; i < nr; ++i) out(i, j) = (*this)(r0 + i, c0 + j);
        return out;
    }
    Mat row(Index i) const { return block_copy(i, 0, 1, c_); }
    Mat col(Index j) const { return block_copy(0, j, r_, 1); }
    Mat leftCols(Index n) const { return block_copy(0, 0, r_, n); }
    Mat topRows(Index n) const { return block_copy(0, 0, n, c_); }

    // ---- reductions (sequential accumulation in storage order)
    T squaredNorm() const {
        T s = T();
        for (const T& v : d_) s += v * v;
        return s;
    }
    T norm() const { return std::sqrt(squaredNorm()); }
    T sum() const {
        T s = T();
        for (const T& v : d_) s += v;
        return s;
    }
    T minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
    T maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
    T dot(const Mat& o) const {
        if (o.size() != size()) shim_detail::fail("dot size");
        T s = T();
        for (Index i = 0; i < size(); ++i) s += d_[static_cast<std::size_t>(i)] * o.d_[static_cast<std::size_t>(i)];
        return s;
    }
    Mat cross(const Mat& o) const {
        if (size() != 3 || o.size() != 3) shim_detail::fail("cross size");
        Mat out(r_, c_);
        const Mat& a = *this;
        out[0] = a[1] * o[2] - a[2] * o[1];
        out[1] = a[2] * o[0] - a[0] * o[2];
        out[2] = a[0] * o[1] - a[1] * o[0];
        return out;
    }
    Mat transpose() const {
        Mat out(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) out(j, i) = (*this)(i, j);
        return out;
    }
    Mat cwiseAbs() const {
        Mat out(r_, c_);
        for (Index i = 0; i < size(); ++i) out[i] = std::abs((*this)[i]);
        return out;
    }

    struct RowwiseOp {
        const Mat& m;
        Mat sum() const {
            Mat out(m.r_, 1);
            for (Index i = 0; i < m.r_; ++i) {
                T s = T();
                for (Index j = 0; j < m.c_; ++j) s += m(i, j);
                out(i, 0) = s;
            }
            return out;
        }
    };
    struct ColwiseOp {
        const Mat& m;
        Mat maxCoeff() const {
            Mat out(1, m.c_);
            for (Index j = 0; j < m.c_; ++j) {
                T s = m(0, j);
                for (Index i = 1; i < m.r_; ++i) s = std::max(s, m(i, j));
                out(0, j) = s;
            }
            return out;
        }
        Mat minCoeff() const {
            Mat out(1, m.c_);
            for (Index j = 0; j < m.c_; ++j) {
                T s = m(0, j);
                for (Index i = 1; i < m.r_; ++i) s = std::min(s, m(i, j));
                out(0, j) = s;
            }
            return out;
        }
    };
    RowwiseOp rowwise() const { return RowwiseOp{*this}; }
    ColwiseOp colwise() const { return ColwiseOp{*this}; }

    JacobiSVD<Mat> jacobiSvd() const;

    // coefficient-wise view (denoise.hpp:221-222, :267)
    struct BoolArray {
        std::vector<char> v;
        bool all() const {
            return std::all_of(v.begin(), v.end(), [](char c) { return c != 0; });
        }
    };
    struct ArrayView {
        const Mat& m;
        Mat sqrt() const {
            Mat out(m.r_, m.c_);
            for (Index i = 0; i < m.size(); ++i) out[i] = std::sqrt(m[i]);
            return out;
        }
        Mat rsqrt() const {
            Mat out(m.r_, m.c_);
            for (Index i = 0; i < m.size(); ++i) out[i] = T(1) / std::sqrt(m[i]);
            return out;
        }
        friend BoolArray operator==(const ArrayView& a, const ArrayView& b) {
            same_shape(a.m, b.m);
            BoolArray out;
            out.v.resize(static_cast<std::size_t>(a.m.size()));
            for (Index i = 0; i < a.m.size(); ++i) out.v[static_cast<std::size_t>(i)] = a.m[i] == b.m[i];
            return out;
        }
    };
    ArrayView array() const { return ArrayView{*this}; }

    // a vector as a (dense, eager) diagonal matrix; inverse() of such a matrix is only
    // used on diagonals (denoise.hpp:225)
    Mat asDiagonal() const {
        const Index n = size();
        Mat out(n, n);
        for (Index i = 0; i < n; ++i) out(i, i) = (*this)[i];
        return out;
    }
    Mat inverse() const {
        if (r_ != c_) shim_detail::fail("inverse of a non-square matrix");
        Mat out(r_, c_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) {
                if (i != j && (*this)(i, j) != T()) shim_detail::fail("inverse(): only diagonal matrices");
                if (i == j) out(i, i) = T(1) / (*this)(i, i);
            }
        return out;
    }

    // ---- arithmetic (hidden friends: found for Mat, its subclasses and BlockRef<Mat>)
    static void same_shape(const Mat& a, const Mat& b) {
        if (a.r_ != b.r_ || a.c_ != b.c_) shim_detail::fail("shape mismatch");
    }
    friend Mat operator+(const Mat& a, const Mat& b) {
        same_shape(a, b);
        Mat out(a.r_, a.c_);
        for (Index i = 0; i < a.size(); ++i) out[i] = a[i] + b[i];
        return out;
    }
    friend Mat operator-(const Mat& a, const Mat& b) {
        same_shape(a, b);
        Mat out(a.r_, a.c_);
        for (Index i = 0; i < a.size(); ++i) out[i] = a[i] - b[i];
        return out;
    }
    friend Mat operator-(const Mat& a) {
        Mat out(a.r_, a.c_);
        for (Index i = 0; i < a.size(); ++i) out[i] = -a[i];
        return out;
    }
    friend Mat operator*(T s, const Mat& a) {
        Mat out(a.r_, a.c_);
        for (Index i = 0; i < a.size(); ++i) out[i] = s * a[i];
        return out;
    }
    friend Mat operator*(const Mat& a, T s) {
        Mat out(a.r_, a.c_);
        for (Index i = 0; i < a.size(); ++i) out[i] = a[i] * s;
        return out;
    }
    friend Mat operator/(const Mat& a, T s) {
        Mat out(a.r_, a.c_);
        for (Index i = 0; i < a.size(); ++i) out[i] = a[i] / s;
        return out;
    }
    // matrix product, accumulated over k in order
    friend Mat operator*(const Mat& a, const Mat& b) {
        if (a.c_ != b.r_) shim_detail::fail("product shape mismatch");
        Mat out(a.r_, b.c_);
        for (Index j = 0; j < b.c_; ++j) {
            T* o = out.data() + j * a.r_;
            for (Index k = 0; k < a.c_; ++k) {
                const T bk = b(k, j);
                const T* ak = a.data() + k * a.r_;
                for (Index i = 0; i < a.r_; ++i) o[i] += ak[i] * bk;
            }
        }
        return out;
    }
    Mat& operator+=(const Mat& o) {
        same_shape(*this, o);
        for (Index i = 0; i < size(); ++i) (*this)[i] += o[i];
        return *this;
    }
    Mat& operator-=(const Mat& o) {
        same_shape(*this, o);
        for (Index i = 0; i < size(); ++i) (*this)[i] -= o[i];
        return *this;
    }
    Mat& operator*=(T s) {
        for (T& v : d_) v *= s;
        return *this;
    }
    Mat& operator/=(T s) {
        for (T& v : d_) v /= s;
        return *this;
    }
};

// Writable view of a rectangular block of a Mat.
template <typename M>
class BlockRef {
    using T = typename M::Scalar;
    M& m_;
    Index r0_, c0_, nr_, nc_;

public:
    BlockRef(M& m, Index r0, Index c0, Index nr, Index nc) : m_(m), r0_(r0), c0_(c0), nr_(nr), nc_(nc) {}
    BlockRef(const BlockRef&) = default;
    Index rows() const { return nr_; }
    Index cols() const { return nc_; }
    Index size() const { return nr_ * nc_; }
    M eval() const { return m_.block_copy(r0_, c0_, nr_, nc_); }
    operator M() const { return eval(); }
    T& operator()(Index i, Index j) { return m_(r0_ + i, c0_ + j); }
    T& operator()(Index i) { return nc_ == 1 ? m_(r0_ + i, c0_) : m_(r0_, c0_ + i); }

    // assignment copies elements; a vector may be assigned to a vector block of
    // the other orientation (Eigen allows that for vectors)
    BlockRef& operator=(const M& src) {
        if (src.rows() == nr_ && src.cols() == nc_) {
            for (Index j = 0; j < nc_; ++j)
                for (Index i = 0; i < nr_; ++i) m_(r0_ + i, c0_ + j) = src(i, j);
        } else if ((nr_ == 1 || nc_ == 1) && (src.rows() == 1 || src.cols() == 1) && src.size() == size()) {
            for (Index i = 0; i < size(); ++i) (*this)(i) = src[i];
        } else {
            shim_detail::fail("block assignment shape mismatch");
        }
        return *this;
    }
    BlockRef& operator=(const BlockRef& o) { return *this = o.eval(); }
    BlockRef& operator+=(const M& o) { return *this = eval() + reshape(o); }
    BlockRef& operator-=(const M& o) { return *this = eval() - reshape(o); }
    BlockRef& operator*=(T s) { return *this = eval() * s; }
    BlockRef& operator/=(T s) { return *this = eval() / s; }
    void setZero() { *this = M(nr_, nc_); }
    void setConstant(T v) {
        M t(nr_, nc_);
        t.setConstant(v);
        *this = t;
    }
    T norm() const { return eval().norm(); }
    T squaredNorm() const { return eval().squaredNorm(); }
    T minCoeff() const { return eval().minCoeff(); }
    T maxCoeff() const { return eval().maxCoeff(); }
    T dot(const M& o) const { return eval().dot(o); }
    M transpose() const { return eval().transpose(); }

private:
    M reshape(const M& o) const {
        if (o.rows() == nr_ && o.cols() == nc_) return o;
        if (o.size() == size() && (o.rows() == 1 || o.cols() == 1)) return o.transpose();
        shim_detail::fail("block arithmetic shape mismatch");
        return o;
    }
};

// The user-facing template: compile-time shape only selects defaults and the
// vector-orientation adaptation on conversion.
template <typename T, int R, int C>
class Matrix : public Mat<T> {
    using B = Mat<T>;
    static constexpr bool kVector = (R == 1 || C == 1);

    void adopt(const B& m) {
        const bool fits = (R == Dynamic || m.rows() == R) && (C == Dynamic || m.cols() == C);
        if (fits) {
            B::operator=(m);
        } else if (kVector && (m.rows() == 1 || m.cols() == 1) && (R == Dynamic || C == Dynamic || m.size() == R * C)) {
            B::operator=(m.transpose());  // a vector of the other orientation
        } else {
            shim_detail::fail("matrix conversion shape mismatch");
        }
    }

public:
    Matrix() : B(R == Dynamic ? 0 : R, C == Dynamic ? 0 : C) {}
    Matrix(Index r, Index c) : B(r, c) {}
    explicit Matrix(Index n) : B(R == 1 ? 1 : n, R == 1 ? n : 1) {}
    Matrix(T x, T y, T z) : B(R == 1 ? 1 : 3, R == 1 ? 3 : 1) {
        (*this)[0] = x;
        (*this)[1] = y;
        (*this)[2] = z;
    }
    Matrix(const B& m) { adopt(m); }
    Matrix(const BlockRef<B>& b) { adopt(b.eval()); }
    Matrix& operator=(const B& m) {
        adopt(m);
        return *this;
    }
    Matrix& operator=(const BlockRef<B>& b) {
        adopt(b.eval());
        return *this;
    }
    using B::resize;
    void resize(Index n) { B::resize(R == 1 ? 1 : n, R == 1 ? n : 1); }

    T& x() { return (*this)[0]; }
    T& y() { return (*this)[1]; }
    T& z() { return (*this)[2]; }
    const T& x() const { return (*this)[0]; }
    const T& y() const { return (*this)[1]; }
    const T& z() const { return (*this)[2]; }

    static Matrix Constant(Index r, Index c, T v) {
        Matrix m(r, c);
        m.setConstant(v);
        return m;
    }
    static Matrix Constant(Index n, T v) {
        Matrix m(n);
        m.setConstant(v);
        return m;
    }
    static Matrix Zero() { return Matrix(); }
    static Matrix Zero(Index n) { return Matrix(n); }
    static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
    static Matrix Ones(Index n) { return Constant(n, T(1)); }
    static Matrix Ones(Index r, Index c) { return Constant(r, c, T(1)); }
    static Matrix Identity(Index r, Index c) {
        Matrix m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = T(1);
        return m;
    }
};

using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using MatrixX3d = Matrix<double, Dynamic, 3>;
using Vector3d = Matrix<double, 3, 1>;
using RowVector3d = Matrix<double, 1, 3>;
using MatrixXi = Matrix<int, Dynamic, Dynamic>;
using VectorXi = Matrix<int, Dynamic, 1>;
using MatrixX3i = Matrix<int, Dynamic, 3>;
using Vector3i = Matrix<int, 3, 1>;

// ---------------------------------------------------------------------------
// HouseholderQR (reference call site spectral.hpp:125-129)
template <typename MatrixType>
class HouseholderQR {
    using T = typename MatrixType::Scalar;
    MatrixType qr_;
    std::vector<T> tau_;

    // H = I - tau v v^T with v = [1; qr_(k+1:, k)], applied to rows k.. of column x
    void apply_reflector(Index k, T* x) const {
        const Index m = qr_.rows();
        const T* v = qr_.data() + k * m;
        T s = x[k];
        for (Index i = k + 1; i < m; ++i) s += v[i] * x[i];
        s *= tau_[static_cast<std::size_t>(k)];
        x[k] -= s;
        for (Index i = k + 1; i < m; ++i) x[i] -= s * v[i];
    }

public:
    explicit HouseholderQR(const Mat<T>& a) : qr_(a) {
        const Index m = qr_.rows(), n = qr_.cols(), steps = std::min(m, n);
        tau_.assign(static_cast<std::size_t>(steps), T());
        for (Index k = 0; k < steps; ++k) {
            T* x = qr_.data() + k * m;
            T tail = T();
            for (Index i = k + 1; i < m; ++i) tail += x[i] * x[i];
            const T c0 = x[k];
            T beta;
            if (tail <= std::numeric_limits<T>::min()) {
                tau_[static_cast<std::size_t>(k)] = T();
                beta = c0;
                for (Index i = k + 1; i < m; ++i) x[i] = T();
            } else {
                beta = std::sqrt(c0 * c0 + tail);
                if (c0 >= T()) beta = -beta;
                const T denom = c0 - beta;
                for (Index i = k + 1; i < m; ++i) x[i] /= denom;
                tau_[static_cast<std::size_t>(k)] = (beta - c0) / beta;
            }
            x[k] = beta;
            for (Index j = k + 1; j < n; ++j) apply_reflector(k, qr_.data() + j * m);
        }
    }
    const MatrixType& matrixQR() const { return qr_; }

    struct Sequence {
        const HouseholderQR& qr;
        // Q * rhs with Q = H_0 H_1 ... H_{steps-1}
        friend MatrixType operator*(const Sequence& s, const Mat<T>& rhs) {
            MatrixType out(rhs);
            const Index steps = static_cast<Index>(s.qr.tau_.size());
            for (Index j = 0; j < out.cols(); ++j)
                for (Index k = steps - 1; k >= 0; --k) s.qr.apply_reflector(k, out.data() + j * out.rows());
            return out;
        }
    };
    Sequence householderQ() const { return Sequence{*this}; }
};

// ---------------------------------------------------------------------------
// SelfAdjointEigenSolver (reference call site spectral.hpp:96): Householder
// tridiagonalisation, eigenvector accumulation, implicit-shift QL.
template <typename MatrixType>
class SelfAdjointEigenSolver {
    using T = typename MatrixType::Scalar;
    Matrix<T, Dynamic, 1> values_;
    MatrixType vectors_;
    ComputationInfo info_ = Success;

public:
    explicit SelfAdjointEigenSolver(const Mat<T>& input) {
        const Index n = input.rows();
        if (input.cols() != n) shim_detail::fail("eigensolver needs a square matrix");
        MatrixType a(input);
        std::vector<T> d(static_cast<std::size_t>(n)), e(static_cast<std::size_t>(n), T());
        std::vector<std::vector<T>> vs(static_cast<std::size_t>(n));  // unit reflector vectors
        std::vector<T> p(static_cast<std::size_t>(n)), w(static_cast<std::size_t>(n));
        // --- reduce to tridiagonal form: A <- H_k A H_k, H_k = I - 2 v v^T on rows k+1..
        for (Index k = 0; k + 2 < n; ++k) {
            const Index m = n - k - 1;
            T* x = a.data() + k * n + (k + 1);
            T nrm2 = T();
            for (Index i = 0; i < m; ++i) nrm2 += x[i] * x[i];
            const T nrm = std::sqrt(nrm2);
            std::vector<T>& v = vs[static_cast<std::size_t>(k)];
            if (nrm2 - x[0] * x[0] <= std::numeric_limits<T>::min()) continue;  // already tridiagonal here
            const T alpha = x[0] >= T() ? -nrm : nrm;
            v.assign(x, x + m);
            v[0] -= alpha;
            T vn = T();
            for (T t : v) vn += t * t;
            vn = std::sqrt(vn);
            for (T& t : v) t /= vn;
            // p = A22 v (A22 = trailing m x m block, full symmetric storage)
            std::fill(p.begin(), p.begin() + m, T());
            for (Index j = 0; j < m; ++j) {
                const T* col = a.data() + (k + 1 + j) * n + (k + 1);
                const T vj = v[static_cast<std::size_t>(j)];
                for (Index i = 0; i < m; ++i) p[static_cast<std::size_t>(i)] += col[i] * vj;
            }
            T kq = T();
            for (Index i = 0; i < m; ++i) kq += v[static_cast<std::size_t>(i)] * p[static_cast<std::size_t>(i)];
            for (Index i = 0; i < m; ++i)
                w[static_cast<std::size_t>(i)] = p[static_cast<std::size_t>(i)] - kq * v[static_cast<std::size_t>(i)];
            // A22 <- A22 - 2 v w^T - 2 w v^T
            for (Index j = 0; j < m; ++j) {
                T* col = a.data() + (k + 1 + j) * n + (k + 1);
                const T vj2 = 2 * v[static_cast<std::size_t>(j)], wj2 = 2 * w[static_cast<std::size_t>(j)];
                for (Index i = 0; i < m; ++i)
                    col[i] -= v[static_cast<std::size_t>(i)] * wj2 + w[static_cast<std::size_t>(i)] * vj2;
            }
            // column / row k of A become (alpha, 0, ..., 0)
            x[0] = alpha;
            for (Index i = 1; i < m; ++i) x[i] = T();
            a(k, k + 1) = alpha;
            for (Index i = 2; i <= m; ++i) a(k, k + i) = T();
        }
        for (Index i = 0; i < n; ++i) d[static_cast<std::size_t>(i)] = a(i, i);
        for (Index i = 0; i + 1 < n; ++i) e[static_cast<std::size_t>(i)] = a(i + 1, i);
        // --- Q = H_0 H_1 ... H_{n-3}
        MatrixType q = MatrixType::Identity(n, n);
        for (Index k = n - 3; k >= 0; --k) {
            const std::vector<T>& v = vs[static_cast<std::size_t>(k)];
            if (v.empty()) continue;
            const Index m = n - k - 1;
            for (Index j = k + 1; j < n; ++j) {
                T* col = q.data() + j * n + (k + 1);
                T s = T();
                for (Index i = 0; i < m; ++i) s += v[static_cast<std::size_t>(i)] * col[i];
                s *= 2;
                for (Index i = 0; i < m; ++i) col[i] -= s * v[static_cast<std::size_t>(i)];
            }
        }
        // --- implicit-shift QL on (d, e); rotations accumulated into q's columns
        for (Index l = 0; l < n; ++l) {
            int iter = 0;
            Index m;
            do {
                for (m = l; m + 1 < n; ++m) {
                    const T dd = std::abs(d[static_cast<std::size_t>(m)]) + std::abs(d[static_cast<std::size_t>(m + 1)]);
                    if (std::abs(e[static_cast<std::size_t>(m)]) <= std::numeric_limits<T>::epsilon() * dd) break;
                }
                if (m != l) {
                    if (iter++ == 60) {
                        info_ = NoConvergence;
                        break;
                    }
                    T g = (d[static_cast<std::size_t>(l + 1)] - d[static_cast<std::size_t>(l)]) /
                          (2 * e[static_cast<std::size_t>(l)]);
                    T r = std::hypot(g, T(1));
                    g = d[static_cast<std::size_t>(m)] - d[static_cast<std::size_t>(l)] +
                        e[static_cast<std::size_t>(l)] / (g + (g >= T() ? std::abs(r) : -std::abs(r)));
                    T s = T(1), c = T(1), pp = T();
                    Index i;
                    for (i = m - 1; i >= l; --i) {
                        T f = s * e[static_cast<std::size_t>(i)];
                        const T b = c * e[static_cast<std::size_t>(i)];
                        r = std::hypot(f, g);
                        e[static_cast<std::size_t>(i + 1)] = r;
                        if (r == T()) {
                            d[static_cast<std::size_t>(i + 1)] -= pp;
                            e[static_cast<std::size_t>(m)] = T();
                            break;
                        }
                        s = f / r;
                        c = g / r;
                        g = d[static_cast<std::size_t>(i + 1)] - pp;
                        r = (d[static_cast<std::size_t>(i)] - g) * s + 2 * c * b;
                        pp = s * r;
                        d[static_cast<std::size_t>(i + 1)] = g + pp;
                        g = c * r - b;
                        T* qi = q.data() + i * n;
                        T* qi1 = q.data() + (i + 1) * n;
                        for (Index k = 0; k < n; ++k) {
                            f = qi1[k];
                            qi1[k] = s * qi[k] + c * f;
                            qi[k] = c * qi[k] - s * f;
                        }
                    }
                    if (r == T() && i >= l) continue;
                    d[static_cast<std::size_t>(l)] -= pp;
                    e[static_cast<std::size_t>(l)] = g;
                    e[static_cast<std::size_t>(m)] = T();
                }
            } while (m != l);
            if (info_ != Success) break;
        }
        // --- ascending order
        std::vector<Index> idx(static_cast<std::size_t>(n));
        std::iota(idx.begin(), idx.end(), Index(0));
        std::stable_sort(idx.begin(), idx.end(),
                         [&](Index x, Index y) { return d[static_cast<std::size_t>(x)] < d[static_cast<std::size_t>(y)]; });
        values_.resize(n);
        vectors_.resize(n, n);
        for (Index j = 0; j < n; ++j) {
            values_(j) = d[static_cast<std::size_t>(idx[static_cast<std::size_t>(j)])];
            std::copy(q.data() + idx[static_cast<std::size_t>(j)] * n, q.data() + (idx[static_cast<std::size_t>(j)] + 1) * n,
                      vectors_.data() + j * n);
        }
    }
    ComputationInfo info() const { return info_; }
    const Matrix<T, Dynamic, 1>& eigenvalues() const { return values_; }
    const MatrixType& eigenvectors() const { return vectors_; }
};

// ---------------------------------------------------------------------------
// JacobiSVD, singular values only (reference call site spectral.hpp:307)
template <typename M>
class JacobiSVD {
    using T = typename M::Scalar;
    Matrix<T, Dynamic, 1> sv_;

public:
    explicit JacobiSVD(const M& input) {
        M a = input.rows() >= input.cols() ? input : input.transpose();
        const Index m = a.rows(), n = a.cols();
        const T eps = std::numeric_limits<T>::epsilon();
        for (int sweep = 0; sweep < 60; ++sweep) {
            bool rotated = false;
            for (Index p = 0; p + 1 < n; ++p)
                for (Index q = p + 1; q < n; ++q) {
                    T* ap = a.data() + p * m;
                    T* aq = a.data() + q * m;
                    T alpha = T(), beta = T(), gamma = T();
                    for (Index i = 0; i < m; ++i) {
                        alpha += ap[i] * ap[i];
                        beta += aq[i] * aq[i];
                        gamma += ap[i] * aq[i];
                    }
                    if (gamma == T() || std::abs(gamma) <= eps * std::sqrt(alpha * beta)) continue;
                    rotated = true;
                    const T zeta = (beta - alpha) / (2 * gamma);
                    const T t = (zeta >= T() ? T(1) : T(-1)) / (std::abs(zeta) + std::sqrt(T(1) + zeta * zeta));
                    const T c = T(1) / std::sqrt(T(1) + t * t), s = c * t;
                    for (Index i = 0; i < m; ++i) {
                        const T x = ap[i], y = aq[i];
                        ap[i] = c * x - s * y;
                        aq[i] = s * x + c * y;
                    }
                }
            if (!rotated) break;
        }
        std::vector<T> s(static_cast<std::size_t>(n));
        for (Index j = 0; j < n; ++j) {
            T v = T();
            for (Index i = 0; i < m; ++i) v += a(i, j) * a(i, j);
            s[static_cast<std::size_t>(j)] = std::sqrt(v);
        }
        std::sort(s.begin(), s.end(), std::greater<T>());
        sv_.resize(n);
        for (Index j = 0; j < n; ++j) sv_(j) = s[static_cast<std::size_t>(j)];
    }
    const Matrix<T, Dynamic, 1>& singularValues() const { return sv_; }
};

template <typename T>
JacobiSVD<Mat<T>> Mat<T>::jacobiSvd() const {
    return JacobiSVD<Mat<T>>(*this);
}

// ---------------------------------------------------------------------------
// Sparse (compressed column) matrix and triplets (spectral.hpp:27, :43-66, :151-154)
template <typename T>
class Triplet {
    Index r_, c_;
    T v_;

public:
    Triplet() : r_(0), c_(0), v_() {}
    Triplet(Index r, Index c, const T& v = T()) : r_(r), c_(c), v_(v) {}
    Index row() const { return r_; }
    Index col() const { return c_; }
    const T& value() const { return v_; }
};

template <typename T>
class SparseMatrix {
    Index r_ = 0, c_ = 0;
    std::vector<int> outer_{0};
    std::vector<int> inner_;
    std::vector<T> val_;

public:
    using Scalar = T;
    SparseMatrix() = default;
    SparseMatrix(Index r, Index c) { resize(r, c); }
    void resize(Index r, Index c) {
        r_ = r;
        c_ = c;
        outer_.assign(static_cast<std::size_t>(c + 1), 0);
        inner_.clear();
        val_.clear();
    }
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index nonZeros() const { return static_cast<Index>(inner_.size()); }
    const int* outerIndexPtr() const { return outer_.data(); }
    const int* innerIndexPtr() const { return inner_.data(); }
    const T* valuePtr() const { return val_.data(); }

    // duplicates are summed; columns come out sorted by row
    template <typename It>
    void setFromTriplets(It first, It last) {
        std::vector<std::vector<std::pair<int, T>>> cols(static_cast<std::size_t>(c_));
        for (It it = first; it != last; ++it)
            cols[static_cast<std::size_t>(it->col())].emplace_back(static_cast<int>(it->row()), it->value());
        outer_.assign(static_cast<std::size_t>(c_ + 1), 0);
        inner_.clear();
        val_.clear();
        for (Index j = 0; j < c_; ++j) {
            auto& col = cols[static_cast<std::size_t>(j)];
            std::stable_sort(col.begin(), col.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
            for (std::size_t i = 0; i < col.size(); ++i) {
                if (!inner_.empty() && static_cast<int>(inner_.size()) > outer_[static_cast<std::size_t>(j)] &&
                    inner_.back() == col[i].first) {
                    val_.back() += col[i].second;
                } else {
                    inner_.push_back(col[i].first);
                    val_.push_back(col[i].second);
                }
            }
            outer_[static_cast<std::size_t>(j + 1)] = static_cast<int>(inner_.size());
        }
    }
    T coeff(Index i, Index j) const {
        const int* b = inner_.data() + outer_[static_cast<std::size_t>(j)];
        const int* e = inner_.data() + outer_[static_cast<std::size_t>(j + 1)];
        const int* it = std::lower_bound(b, e, static_cast<int>(i));
        return (it != e && *it == i) ? val_[static_cast<std::size_t>(it - inner_.data())] : T();
    }
    void setIdentity() {
        const Index n = std::min(r_, c_);
        outer_.assign(static_cast<std::size_t>(c_ + 1), 0);
        inner_.clear();
        val_.clear();
        for (Index j = 0; j < c_; ++j) {
            if (j < n) {
                inner_.push_back(static_cast<int>(j));
                val_.push_back(T(1));
            }
            outer_[static_cast<std::size_t>(j + 1)] = static_cast<int>(inner_.size());
        }
    }
    friend SparseMatrix operator*(T s, const SparseMatrix& a) {
        SparseMatrix out = a;
        for (T& v : out.val_) v = s * v;
        return out;
    }
    SparseMatrix& operator+=(const SparseMatrix& o) {
        if (o.r_ != r_ || o.c_ != c_) shim_detail::fail("sparse shape mismatch");
        std::vector<int> outer(static_cast<std::size_t>(c_ + 1), 0), inner;
        std::vector<T> val;
        for (Index j = 0; j < c_; ++j) {
            int a = outer_[static_cast<std::size_t>(j)], ae = outer_[static_cast<std::size_t>(j + 1)];
            int b = o.outer_[static_cast<std::size_t>(j)], be = o.outer_[static_cast<std::size_t>(j + 1)];
            while (a < ae || b < be) {
                if (b >= be || (a < ae && inner_[static_cast<std::size_t>(a)] < o.inner_[static_cast<std::size_t>(b)])) {
                    inner.push_back(inner_[static_cast<std::size_t>(a)]);
                    val.push_back(val_[static_cast<std::size_t>(a++)]);
                } else if (a >= ae || o.inner_[static_cast<std::size_t>(b)] < inner_[static_cast<std::size_t>(a)]) {
                    inner.push_back(o.inner_[static_cast<std::size_t>(b)]);
                    val.push_back(o.val_[static_cast<std::size_t>(b++)]);
                } else {
                    inner.push_back(inner_[static_cast<std::size_t>(a)]);
                    val.push_back(val_[static_cast<std::size_t>(a++)] + o.val_[static_cast<std::size_t>(b++)]);
                }
            }
            outer[static_cast<std::size_t>(j + 1)] = static_cast<int>(inner.size());
        }
        outer_.swap(outer);
        inner_.swap(inner);
        val_.swap(val);
        return *this;
    }
    operator Mat<T>() const {
        Mat<T> out(r_, c_);
        for (Index j = 0; j < c_; ++j)
            for (int k = outer_[static_cast<std::size_t>(j)]; k < outer_[static_cast<std::size_t>(j + 1)]; ++k)
                out(inner_[static_cast<std::size_t>(k)], j) = val_[static_cast<std::size_t>(k)];
        return out;
    }
};

// ---------------------------------------------------------------------------
// SimplicialLDLT (reference call sites spectral.hpp:155-156, :168, :174):
// P A P^T = L D L^T on the envelope of the reverse Cuthill-McKee ordered matrix,
// no pivoting (an indefinite matrix is tolerated, a zero pivot is not).
template <typename SparseType>
class SimplicialLDLT {
    using T = typename SparseType::Scalar;
    Index n_ = 0;
    std::vector<int> perm_;            // new index -> old index
    std::vector<int> first_;           // first column of row i's envelope
    std::vector<std::size_t> start_;   // offset of row i's envelope in l_
    std::vector<T> l_, d_;
    ComputationInfo info_ = InvalidInput;

    static std::vector<int> rcm(const SparseType& a) {
        const int n = static_cast<int>(a.rows());
        const int* op = a.outerIndexPtr();
        const int* ip = a.innerIndexPtr();
        auto degree = [&](int v) { return op[v + 1] - op[v]; };
        std::vector<int> order;
        order.reserve(static_cast<std::size_t>(n));
        std::vector<char> seen(static_cast<std::size_t>(n), 0);
        std::vector<int> level(static_cast<std::size_t>(n));
        auto bfs_last = [&](int s, std::vector<int>& visited) {
            // BFS from s over unseen vertices; returns a minimum-degree vertex of the last level
            visited.clear();
            visited.push_back(s);
            level[static_cast<std::size_t>(s)] = 0;
            std::vector<char> mark(static_cast<std::size_t>(n), 0);
            mark[static_cast<std::size_t>(s)] = 1;
            for (std::size_t h = 0; h < visited.size(); ++h) {
                const int v = visited[h];
                for (int k = op[v]; k < op[v + 1]; ++k) {
                    const int w = ip[k];
                    if (w == v || seen[static_cast<std::size_t>(w)] || mark[static_cast<std::size_t>(w)]) continue;
                    mark[static_cast<std::size_t>(w)] = 1;
                    level[static_cast<std::size_t>(w)] = level[static_cast<std::size_t>(v)] + 1;
                    visited.push_back(w);
                }
            }
            const int last = level[static_cast<std::size_t>(visited.back())];
            int best = visited.back();
            for (int v : visited)
                if (level[static_cast<std::size_t>(v)] == last && degree(v) < degree(best)) best = v;
            return best;
        };
        std::vector<int> comp;
        for (int root = 0; root < n; ++root) {
            if (seen[static_cast<std::size_t>(root)]) continue;
            int s = root;
            for (int rep = 0; rep < 3; ++rep) s = bfs_last(s, comp);  // pseudo-peripheral start
            // Cuthill-McKee from s, neighbours by ascending degree
            const std::size_t base = order.size();
            order.push_back(s);
            seen[static_cast<std::size_t>(s)] = 1;
            for (std::size_t h = base; h < order.size(); ++h) {
                const int v = order[h];
                std::vector<int> nb;
                for (int k = op[v]; k < op[v + 1]; ++k) {
                    const int w = ip[k];
                    if (w != v && !seen[static_cast<std::size_t>(w)]) {
                        seen[static_cast<std::size_t>(w)] = 1;
                        nb.push_back(w);
                    }
                }
                std::stable_sort(nb.begin(), nb.end(), [&](int x, int y) { return degree(x) < degree(y); });
                order.insert(order.end(), nb.begin(), nb.end());
            }
        }
        std::reverse(order.begin(), order.end());
        return order;
    }

public:
    SimplicialLDLT() = default;
    void compute(const SparseType& a) {
        n_ = a.rows();
        if (a.cols() != n_) {
            info_ = InvalidInput;
            return;
        }
        const int n = static_cast<int>(n_);
        perm_ = rcm(a);
        std::vector<int> inv(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) inv[static_cast<std::size_t>(perm_[static_cast<std::size_t>(i)])] = i;
        const int* op = a.outerIndexPtr();
        const int* ip = a.innerIndexPtr();
        const T* vp = a.valuePtr();
        first_.assign(static_cast<std::size_t>(n), 0);
        for (int i = 0; i < n; ++i) {
            const int old = perm_[static_cast<std::size_t>(i)];
            int f = i;
            for (int k = op[old]; k < op[old + 1]; ++k) f = std::min(f, inv[static_cast<std::size_t>(ip[k])]);
            first_[static_cast<std::size_t>(i)] = f;
        }
        start_.assign(static_cast<std::size_t>(n + 1), 0);
        for (int i = 0; i < n; ++i)
            start_[static_cast<std::size_t>(i + 1)] =
                start_[static_cast<std::size_t>(i)] + static_cast<std::size_t>(i - first_[static_cast<std::size_t>(i)]);
        l_.assign(start_[static_cast<std::size_t>(n)], T());
        d_.assign(static_cast<std::size_t>(n), T());
        for (int i = 0; i < n; ++i) {
            const int old = perm_[static_cast<std::size_t>(i)];
            T* row = l_.data() + start_[static_cast<std::size_t>(i)] - first_[static_cast<std::size_t>(i)];
            for (int k = op[old]; k < op[old + 1]; ++k) {
                const int j = inv[static_cast<std::size_t>(ip[k])];
                if (j < i) row[j] = vp[k];
                else if (j == i) d_[static_cast<std::size_t>(i)] = vp[k];
            }
        }
        info_ = Success;
        // row by row: w_j = a_ij - sum_{k<j} w_k L_jk ; L_ij = w_j / d_j ; d_i = a_ii - sum_j w_j L_ij
        for (int i = 0; i < n; ++i) {
            const int fi = first_[static_cast<std::size_t>(i)];
            T* wi = l_.data() + start_[static_cast<std::size_t>(i)] - fi;
            for (int j = fi; j < i; ++j) {
                const int fj = first_[static_cast<std::size_t>(j)];
                const T* lj = l_.data() + start_[static_cast<std::size_t>(j)] - fj;
                T s = wi[j];
                for (int k = std::max(fi, fj); k < j; ++k) s -= wi[k] * lj[k];
                wi[j] = s;
            }
            T di = d_[static_cast<std::size_t>(i)];
            for (int j = fi; j < i; ++j) {
                const T w = wi[j];
                wi[j] = w / d_[static_cast<std::size_t>(j)];
                di -= w * wi[j];
            }
            d_[static_cast<std::size_t>(i)] = di;
            if (di == T() || !std::isfinite(di)) {
                info_ = NumericalIssue;
                return;
            }
        }
    }
    ComputationInfo info() const { return info_; }

    Matrix<T, Dynamic, Dynamic> solve(const Mat<T>& b) const {
        const Index n = n_, c = b.cols();
        if (b.rows() != n) shim_detail::fail("solve shape mismatch");
        std::vector<T> x(static_cast<std::size_t>(n * c));  // row-major, permuted rows
        for (Index i = 0; i < n; ++i) {
            const Index old = perm_[static_cast<std::size_t>(i)];
            for (Index j = 0; j < c; ++j) x[static_cast<std::size_t>(i * c + j)] = b(old, j);
        }
        for (Index i = 0; i < n; ++i) {  // L y = b
            const int fi = first_[static_cast<std::size_t>(i)];
            const T* li = l_.data() + start_[static_cast<std::size_t>(i)] - fi;
            T* xi = x.data() + i * c;
            for (Index j = fi; j < i; ++j) {
                const T lij = li[j];
                const T* xj = x.data() + j * c;
                for (Index k = 0; k < c; ++k) xi[k] -= lij * xj[k];
            }
        }
        for (Index i = 0; i < n; ++i) {
            const T di = d_[static_cast<std::size_t>(i)];
            T* xi = x.data() + i * c;
            for (Index k = 0; k < c; ++k) xi[k] /= di;
        }
        for (Index i = n - 1; i >= 0; --i) {  // L^T x = y
            const int fi = first_[static_cast<std::size_t>(i)];
            const T* li = l_.data() + start_[static_cast<std::size_t>(i)] - fi;
            const T* xi = x.data() + i * c;
            for (Index j = fi; j < i; ++j) {
                const T lij = li[j];
                T* xj = x.data() + j * c;
                for (Index k = 0; k < c; ++k) xj[k] -= lij * xi[k];
            }
        }
        Matrix<T, Dynamic, Dynamic> out(n, c);
        for (Index i = 0; i < n; ++i) {
            const Index old = perm_[static_cast<std::size_t>(i)];
            for (Index j = 0; j < c; ++j) out(old, j) = x[static_cast<std::size_t>(i * c + j)];
        }
        return out;
    }
};

}  // namespace Eigen
