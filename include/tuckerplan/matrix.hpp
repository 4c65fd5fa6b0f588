// tuckerplan (B200 engine) : minimal column-major matrix.
// The reference's signatures take Eigen::MatrixXd (ttm.hpp:43-73, hooi.hpp:39-81).  Eigen is not a dependency of
// this engine; `Matrix` has the same storage (column-major, leading dimension = rows) and the accessors the
// reference API relies on.  Every function that takes a matrix here is a template over "anything with
// rows(), cols() and operator()(i, j)", so Eigen matrices and expressions (e.g. `F.transpose()`) are accepted
// unchanged when the caller does have Eigen.
#pragma once

#include <cstddef>
#include <vector>

namespace tuckerplan {

class Matrix {
 public:
  Matrix() = default;
  Matrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), data_(rows * cols, 0.0) {}
  static Matrix Zero(std::size_t rows, std::size_t cols) { return Matrix(rows, cols); }
  static Matrix Identity(std::size_t rows, std::size_t cols) {
    Matrix m(rows, cols);
    for (std::size_t i = 0; i < rows && i < cols; ++i) m(i, i) = 1.0;
    return m;
  }
  template <class Other>
  static Matrix from(const Other& o) {  // copy from any rows()/cols()/(i,j) type
    Matrix m(static_cast<std::size_t>(o.rows()), static_cast<std::size_t>(o.cols()));
    for (std::size_t j = 0; j < m.cols_; ++j)
      for (std::size_t i = 0; i < m.rows_; ++i) m(i, j) = o(i, j);
    return m;
  }
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  std::size_t size() const { return data_.size(); }
  double& operator()(std::size_t i, std::size_t j) { return data_[j * rows_ + i]; }
  double operator()(std::size_t i, std::size_t j) const { return data_[j * rows_ + i]; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  Matrix transpose() const {
    Matrix t(cols_, rows_);
    for (std::size_t j = 0; j < cols_; ++j)
      for (std::size_t i = 0; i < rows_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  bool operator==(const Matrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_ && data_ == o.data_; }

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

using MatrixXd = Matrix;  // the name the reference signatures use, inside namespace tuckerplan

namespace detail {
// Column-major copy of any matrix-like argument (no copy when it already is a Matrix).
inline const Matrix& as_matrix(const Matrix& m, Matrix&) { return m; }
template <class Other>
const Matrix& as_matrix(const Other& o, Matrix& scratch) {
  scratch = Matrix::from(o);
  return scratch;
}
}  // namespace detail

}  // namespace tuckerplan
