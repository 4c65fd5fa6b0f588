// Seeded host-side inputs with the reference's streams: a 64-bit Mersenne
// twister feeding ONE std::normal_distribution<double> object (whose cached
// second variate carries across calls), reference dense_tensor.hpp:43-49 and
// hooi.hpp:109-120.  The draw sequence is libstdc++'s; this library is built
// with the same toolchain as the reference would be.
#pragma once

#include <cmath>
#include <cstddef>
#include <random>
#include <vector>

#include "common.hpp"

namespace tpb {

class GaussianStream {
 public:
  explicit GaussianStream(u64 seed) : engine_(seed), normal_(0.0, 1.0) {}
  double next() { return normal_(engine_); }
  void fill(double* out, std::size_t n) {
    for (std::size_t i = 0; i < n; ++i) out[i] = normal_(engine_);
  }

 private:
  std::mt19937_64 engine_;
  std::normal_distribution<double> normal_;
};

// Thin Q (rows x cols, column-major, ld = rows) of the Householder QR of the
// column-major matrix `a` (overwritten).  Reflector convention of Eigen's
// HouseholderQR / LAPACK dgeqr2+dorg2r: beta = -sign(alpha) * ||x||,
// tau = (beta - alpha) / beta, v = [1; x_tail / (alpha - beta)]; Q = H_0 ... H_{k-1}.
inline void householder_thin_q(double* a, std::size_t rows, std::size_t cols, double* q) {
  const std::size_t k = cols < rows ? cols : rows;
  std::vector<double> tau(k, 0.0);
  for (std::size_t j = 0; j < k; ++j) {
    double* col = a + j * rows;
    double tail = 0.0;
    for (std::size_t i = j + 1; i < rows; ++i) tail += col[i] * col[i];
    const double alpha = col[j];
    if (tail == 0.0) {
      tau[j] = 0.0;  // H = I (Eigen: tailSqNorm <= tiny -> tau = 0, beta = alpha)
    } else {
      double beta = std::sqrt(alpha * alpha + tail);
      if (alpha >= 0.0) beta = -beta;
      tau[j] = (beta - alpha) / beta;
      const double scale = 1.0 / (alpha - beta);
      for (std::size_t i = j + 1; i < rows; ++i) col[i] *= scale;
      col[j] = beta;
      // apply H_j = I - tau v v^T to the trailing columns
      for (std::size_t c = j + 1; c < cols; ++c) {
        double* other = a + c * rows;
        double dot = other[j];
        for (std::size_t i = j + 1; i < rows; ++i) dot += col[i] * other[i];
        dot *= tau[j];
        other[j] -= dot;
        for (std::size_t i = j + 1; i < rows; ++i) other[i] -= dot * col[i];
      }
    }
  }
  // Q = H_0 ... H_{k-1} applied to the first `cols` columns of the identity, back to front
  for (std::size_t c = 0; c < cols; ++c)
    for (std::size_t i = 0; i < rows; ++i) q[c * rows + i] = (i == c) ? 1.0 : 0.0;
  for (std::size_t jj = k; jj-- > 0;) {
    const double* v = a + jj * rows;  // v[jj] is implicitly 1
    if (tau[jj] == 0.0) continue;
    for (std::size_t c = 0; c < cols; ++c) {
      double* qc = q + c * rows;
      double dot = qc[jj];
      for (std::size_t i = jj + 1; i < rows; ++i) dot += v[i] * qc[i];
      dot *= tau[jj];
      qc[jj] -= dot;
      for (std::size_t i = jj + 1; i < rows; ++i) qc[i] -= dot * v[i];
    }
  }
}

}  // namespace tpb
