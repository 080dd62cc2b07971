// Small dense fp64 linear algebra for the one-time host precompute of fdtd_add_rom.
// Row-major storage.  Sizes are the ROM orders (<= a few hundred).
#pragma once
#include <cmath>
#include <cstdint>
#include <vector>

namespace fdtd {
namespace dense {

using Mat = std::vector<double>;

inline Mat zeros(int r, int c) { return Mat((size_t)r * c, 0.0); }

// C(m x n) = A(m x k) B(k x n)
inline Mat matmul(const Mat& A, const Mat& B, int m, int k, int n) {
  Mat C = zeros(m, n);
  for (int i = 0; i < m; ++i)
    for (int l = 0; l < k; ++l) {
      const double a = A[(size_t)i * k + l];
      if (a == 0.0) continue;
      for (int j = 0; j < n; ++j) C[(size_t)i * n + j] += a * B[(size_t)l * n + j];
    }
  return C;
}

inline Mat transpose(const Mat& A, int m, int n) {
  Mat T = zeros(n, m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) T[(size_t)j * m + i] = A[(size_t)i * n + j];
  return T;
}

// Inverse by LU with partial pivoting (Gauss-Jordan on [A | I]).  Returns false if singular.
inline bool inverse(const Mat& A, int n, Mat& out) {
  Mat M = A;
  out = zeros(n, n);
  for (int i = 0; i < n; ++i) out[(size_t)i * n + i] = 1.0;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::fabs(M[(size_t)k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      const double v = std::fabs(M[(size_t)i * n + k]);
      if (v > best) { best = v; p = i; }
    }
    if (!(best > 0.0)) return false;
    if (p != k)
      for (int j = 0; j < n; ++j) {
        std::swap(M[(size_t)k * n + j], M[(size_t)p * n + j]);
        std::swap(out[(size_t)k * n + j], out[(size_t)p * n + j]);
      }
    const double inv = 1.0 / M[(size_t)k * n + k];
    for (int j = 0; j < n; ++j) { M[(size_t)k * n + j] *= inv; out[(size_t)k * n + j] *= inv; }
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double f = M[(size_t)i * n + k];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        M[(size_t)i * n + j] -= f * M[(size_t)k * n + j];
        out[(size_t)i * n + j] -= f * out[(size_t)k * n + j];
      }
    }
  }
  return true;
}

// In-place Cholesky test of a symmetric matrix: true iff positive definite.
inline bool cholesky_ok(Mat A, int n) {
  for (int j = 0; j < n; ++j) {
    double d = A[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= A[(size_t)j * n + k] * A[(size_t)j * n + k];
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    A[(size_t)j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double s = A[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
      A[(size_t)i * n + j] = s / d;
    }
  }
  return true;
}

}  // namespace dense
}  // namespace fdtd
