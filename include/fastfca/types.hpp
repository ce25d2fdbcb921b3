// types.hpp -- scalar and dense-matrix types of the FastFCA C++ API
// (drop-in for reference proj/include/fastfca/types.hpp:13-24).
//
// With Eigen available the aliases are the reference's (Eigen::MatrixXcd, ...),
// so code written against the reference compiles unchanged.  Without Eigen
// (this image) a minimal column-major dense matrix with the same element
// layout stands in: element (r, c) at data()[r + c * rows()].
#pragma once

#include <algorithm>
#include <complex>
#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>

#if defined(FFCA_USE_EIGEN) || (defined(__has_include) && __has_include(<Eigen/Dense>) && !defined(FFCA_NO_EIGEN))
#include <Eigen/Dense>
#define FFCA_HAVE_EIGEN 1
#endif

namespace fastfca {

using Complex = std::complex<double>;

#ifdef FFCA_HAVE_EIGEN
using CMat = Eigen::MatrixXcd;
using CVec = Eigen::VectorXcd;
using RMat = Eigen::MatrixXd;
using RVec = Eigen::VectorXd;
#else
// Column-major dense matrix (Eigen's default storage order).
template <typename T>
class Dense {
 public:
  Dense() = default;
  Dense(long rows, long cols) : r_(rows), c_(cols), a_(size_t(rows * cols), T(0)) {}
  explicit Dense(long n) : Dense(n, 1) {}  // column vector (Eigen::VectorX*(n))
  static Dense Zero(long rows, long cols) { return Dense(rows, cols); }
  static Dense Zero(long n) { return Dense(n, 1); }
  static Dense Ones(long rows, long cols) {
    Dense m(rows, cols);
    std::fill(m.a_.begin(), m.a_.end(), T(1));
    return m;
  }
  static Dense Constant(long rows, long cols, T v) {
    Dense m(rows, cols);
    std::fill(m.a_.begin(), m.a_.end(), v);
    return m;
  }
  static Dense Identity(long rows, long cols) {
    Dense m(rows, cols);
    for (long k = 0; k < std::min(rows, cols); ++k) m(k, k) = T(1);
    return m;
  }
  long rows() const { return r_; }
  long cols() const { return c_; }
  long size() const { return r_ * c_; }
  void resize(long rows, long cols) {
    r_ = rows, c_ = cols;
    a_.assign(size_t(rows * cols), T(0));
  }
  T& operator()(long r, long c) { return a_[size_t(r + c * r_)]; }
  const T& operator()(long r, long c) const { return a_[size_t(r + c * r_)]; }
  T& operator()(long k) { return a_[size_t(k)]; }
  const T& operator()(long k) const { return a_[size_t(k)]; }
  T* data() { return a_.data(); }
  const T* data() const { return a_.data(); }

 private:
  long r_ = 0, c_ = 0;
  std::vector<T> a_;
};
using CMat = Dense<Complex>;
using CVec = Dense<Complex>;
using RMat = Dense<double>;
using RVec = Dense<double>;
#endif

// Unrecoverable numerical condition (singular reduction, non-finite update);
// reference types.hpp:21-24.
class NumericalError : public std::runtime_error {
 public:
  explicit NumericalError(const std::string& what) : std::runtime_error(what) {}
};

}  // namespace fastfca
