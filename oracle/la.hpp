// ORACLE — test infrastructure only.  A CPU restatement of the reference
// heterodyn solver (/root/reference/proj/src) used as the parity checker and
// the timed CPU baseline.  Nothing in the product package may link or call it.
//
// Small dense linear algebra that replaces the Eigen calls of the reference.
// Eigen is not installed here, so its algorithms are restated:
//   * JacobiSVD<Matrix3d> (two-sided Jacobi; used by signed_svd,
//     localstep.cpp:99-114) mirrors Eigen's sweep order, 2x2 real SVD and
//     final sign/sort steps so U/V conventions agree in the generic case;
//   * SelfAdjointEigenSolver<Matrix3d> (localstep.cpp:49,294,361,413) is a
//     cyclic Jacobi eigen-solver (ascending eigenvalues; callers only use
//     convention-invariant products);
//   * LDLT<MatrixXd> (forward.cpp:42, contact.cpp:248, backward.cpp:261) is a
//     diagonal-pivoting LDL^T like Eigen's;
//   * FullPivLU<Matrix4d> (localstep.cpp:215,395) is complete-pivoting LU.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <vector>

namespace hdo {

using Scalar = double;

struct Vec3 {
  double v[3] = {0, 0, 0};
  Vec3() = default;
  Vec3(double a, double b, double c) { v[0] = a; v[1] = b; v[2] = c; }
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
  static Vec3 ones() { return Vec3(1, 1, 1); }
  double dot(const Vec3& o) const { return v[0] * o.v[0] + v[1] * o.v[1] + v[2] * o.v[2]; }
  double squaredNorm() const { return dot(*this); }
  double norm() const { return std::sqrt(squaredNorm()); }
  double prod() const { return v[0] * v[1] * v[2]; }
  Vec3 operator+(const Vec3& o) const { return Vec3(v[0] + o.v[0], v[1] + o.v[1], v[2] + o.v[2]); }
  Vec3 operator-(const Vec3& o) const { return Vec3(v[0] - o.v[0], v[1] - o.v[1], v[2] - o.v[2]); }
  Vec3 operator*(double s) const { return Vec3(v[0] * s, v[1] * s, v[2] * s); }
  Vec3 operator/(double s) const { return Vec3(v[0] / s, v[1] / s, v[2] / s); }
  Vec3& operator+=(const Vec3& o) { for (int i = 0; i < 3; ++i) v[i] += o.v[i]; return *this; }
  Vec3& operator-=(const Vec3& o) { for (int i = 0; i < 3; ++i) v[i] -= o.v[i]; return *this; }
  Vec3 cross(const Vec3& o) const {
    return Vec3(v[1] * o.v[2] - v[2] * o.v[1], v[2] * o.v[0] - v[0] * o.v[2],
                v[0] * o.v[1] - v[1] * o.v[0]);
  }
  Vec3 cwiseAbs() const { return Vec3(std::fabs(v[0]), std::fabs(v[1]), std::fabs(v[2])); }
  Vec3 cwiseMax(double s) const { return Vec3(std::max(v[0], s), std::max(v[1], s), std::max(v[2], s)); }
  double maxCoeff() const { return std::max(v[0], std::max(v[1], v[2])); }
  double minCoeff() const { return std::min(v[0], std::min(v[1], v[2])); }
};
inline Vec3 operator*(double s, const Vec3& a) { return a * s; }

// Column-major 3x3 (vec(F)[3c + r] = F(r, c), as Eigen's storage).
struct Mat3 {
  double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double& operator()(int r, int c) { return m[r + 3 * c]; }
  double operator()(int r, int c) const { return m[r + 3 * c]; }
  static Mat3 identity() { Mat3 a; a.m[0] = a.m[4] = a.m[8] = 1; return a; }
  static Mat3 diag(const Vec3& d) { Mat3 a; a.m[0] = d[0]; a.m[4] = d[1]; a.m[8] = d[2]; return a; }
  Vec3 col(int c) const { return Vec3(m[3 * c], m[3 * c + 1], m[3 * c + 2]); }
  void set_col(int c, const Vec3& x) { m[3 * c] = x[0]; m[3 * c + 1] = x[1]; m[3 * c + 2] = x[2]; }
  Vec3 row(int r) const { return Vec3(m[r], m[r + 3], m[r + 6]); }
  Mat3 transpose() const {
    Mat3 t;
    for (int r = 0; r < 3; ++r) for (int c = 0; c < 3; ++c) t(c, r) = (*this)(r, c);
    return t;
  }
  Mat3 operator*(const Mat3& b) const {
    Mat3 o;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double s = 0;
        for (int k = 0; k < 3; ++k) s += (*this)(r, k) * b(k, c);
        o(r, c) = s;
      }
    return o;
  }
  Vec3 operator*(const Vec3& x) const {
    Vec3 o;
    for (int r = 0; r < 3; ++r) o[r] = (*this)(r, 0) * x[0] + (*this)(r, 1) * x[1] + (*this)(r, 2) * x[2];
    return o;
  }
  Mat3 operator+(const Mat3& b) const { Mat3 o; for (int i = 0; i < 9; ++i) o.m[i] = m[i] + b.m[i]; return o; }
  Mat3 operator-(const Mat3& b) const { Mat3 o; for (int i = 0; i < 9; ++i) o.m[i] = m[i] - b.m[i]; return o; }
  Mat3 operator*(double s) const { Mat3 o; for (int i = 0; i < 9; ++i) o.m[i] = m[i] * s; return o; }
  double squaredNorm() const { double s = 0; for (double x : m) s += x * x; return s; }
  double norm() const { return std::sqrt(squaredNorm()); }
  // Eigen's 3x3 cofactor expansion along the first column.
  double determinant() const {
    const Mat3& a = *this;
    return a(0, 0) * (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) -
           a(1, 0) * (a(0, 1) * a(2, 2) - a(0, 2) * a(2, 1)) +
           a(2, 0) * (a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1));
  }
  Mat3 inverse() const {
    const Mat3& a = *this;
    Mat3 cof;
    cof(0, 0) = a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1);
    cof(1, 0) = a(1, 2) * a(2, 0) - a(1, 0) * a(2, 2);
    cof(2, 0) = a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0);
    const double det = cof(0, 0) * a(0, 0) + cof(1, 0) * a(0, 1) + cof(2, 0) * a(0, 2);
    const double inv = 1.0 / det;
    Mat3 r;
    r(0, 0) = cof(0, 0) * inv;
    r(0, 1) = (a(0, 2) * a(2, 1) - a(0, 1) * a(2, 2)) * inv;
    r(0, 2) = (a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1)) * inv;
    r(1, 0) = cof(1, 0) * inv;
    r(1, 1) = (a(0, 0) * a(2, 2) - a(0, 2) * a(2, 0)) * inv;
    r(1, 2) = (a(0, 2) * a(1, 0) - a(0, 0) * a(1, 2)) * inv;
    r(2, 0) = cof(2, 0) * inv;
    r(2, 1) = (a(0, 1) * a(2, 0) - a(0, 0) * a(2, 1)) * inv;
    r(2, 2) = (a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0)) * inv;
    return r;
  }
};
inline Mat3 operator*(double s, const Mat3& a) { return a * s; }
inline Mat3 outer(const Vec3& a, const Vec3& b) {
  Mat3 o;
  for (int r = 0; r < 3; ++r) for (int c = 0; c < 3; ++c) o(r, c) = a[r] * b[c];
  return o;
}

// ---- JacobiSVD<Matrix3d> restatement --------------------------------------
// Plane rotation (c, s) with Eigen's JacobiRotation semantics.
struct Rot { double c = 1, s = 0; };
inline Rot rot_mul(const Rot& a, const Rot& b) { return {a.c * b.c - a.s * b.s, a.c * b.s + a.s * b.c}; }
inline Rot rot_t(const Rot& a) { return {a.c, -a.s}; }
// apply_rotation_in_the_plane(x, y, j): x' = c x + s y, y' = -s x + c y.
inline void rot_rows(Mat3& m, int p, int q, const Rot& j) {
  for (int i = 0; i < 3; ++i) {
    const double xi = m(p, i), yi = m(q, i);
    m(p, i) = j.c * xi + j.s * yi;
    m(q, i) = -j.s * xi + j.c * yi;
  }
}
// applyOnTheRight(p, q, j) == apply_rotation_in_the_plane(col p, col q, j^T).
inline void rot_cols_right(Mat3& m, int p, int q, const Rot& j) {
  const Rot t = rot_t(j);
  for (int i = 0; i < 3; ++i) {
    const double xi = m(i, p), yi = m(i, q);
    m(i, p) = t.c * xi + t.s * yi;
    m(i, q) = -t.s * xi + t.c * yi;
  }
}
inline bool make_jacobi(double x, double y, double z, Rot& r) {
  const double deno = 2.0 * std::fabs(y);
  if (deno < DBL_MIN) { r.c = 1; r.s = 0; return false; }
  const double tau = (x - z) / deno;
  const double w = std::sqrt(tau * tau + 1.0);
  const double t = tau > 0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
  const double sign_t = t > 0 ? 1.0 : -1.0;
  const double n = 1.0 / std::sqrt(t * t + 1.0);
  r.s = -sign_t * (y / std::fabs(y)) * std::fabs(t) * n;
  r.c = n;
  return true;
}
inline void real_2x2_jacobi_svd(const Mat3& w, int p, int q, Rot& jl, Rot& jr) {
  double m00 = w(p, p), m01 = w(p, q), m10 = w(q, p), m11 = w(q, q);
  Rot r1;
  const double t = m00 + m11, d = m10 - m01;
  if (std::fabs(d) < DBL_MIN) { r1.s = 0; r1.c = 1; }
  else { const double u = t / d; const double tmp = std::sqrt(1.0 + u * u); r1.s = 1.0 / tmp; r1.c = u / tmp; }
  const double n00 = r1.c * m00 + r1.s * m10, n01 = r1.c * m01 + r1.s * m11;
  const double n11 = -r1.s * m01 + r1.c * m11;
  make_jacobi(n00, n01, n11, jr);
  jl = rot_mul(r1, rot_t(jr));
}
inline void jacobi_svd3(const Mat3& a, Mat3& u, Vec3& sig, Mat3& v) {
  double scale = 0;
  for (double x : a.m) scale = std::max(scale, std::fabs(x));
  if (scale == 0) scale = 1;
  Mat3 w;
  for (int i = 0; i < 9; ++i) w.m[i] = a.m[i] / scale;
  u = Mat3::identity();
  v = Mat3::identity();
  const double precision = 2.0 * DBL_EPSILON;
  double max_diag = std::max(std::fabs(w(0, 0)), std::max(std::fabs(w(1, 1)), std::fabs(w(2, 2))));
  bool finished = false;
  int sweeps = 0;
  while (!finished && sweeps < 100) {
    finished = true;
    ++sweeps;
    for (int p = 1; p < 3; ++p)
      for (int q = 0; q < p; ++q) {
        const double threshold = std::max(DBL_MIN, precision * max_diag);
        if (std::fabs(w(p, q)) > threshold || std::fabs(w(q, p)) > threshold) {
          finished = false;
          Rot jl, jr;
          real_2x2_jacobi_svd(w, p, q, jl, jr);
          rot_rows(w, p, q, jl);
          rot_cols_right(u, p, q, rot_t(jl));
          rot_cols_right(w, p, q, jr);
          rot_cols_right(v, p, q, jr);
          max_diag = std::max(max_diag, std::max(std::fabs(w(p, p)), std::fabs(w(q, q))));
        }
      }
  }
  for (int i = 0; i < 3; ++i) {
    const double d = w(i, i);
    sig[i] = std::fabs(d);
    if (d < 0) u.set_col(i, u.col(i) * -1.0);
  }
  sig = sig * scale;
  for (int i = 0; i < 3; ++i) {
    int pos = i;
    double best = sig[i];
    for (int k = i + 1; k < 3; ++k)
      if (sig[k] > best) { best = sig[k]; pos = k; }
    if (best == 0) break;
    if (pos != i) {
      std::swap(sig[i], sig[pos]);
      const Vec3 ui = u.col(i), up = u.col(pos);
      u.set_col(i, up); u.set_col(pos, ui);
      const Vec3 vi = v.col(i), vp = v.col(pos);
      v.set_col(i, vp); v.set_col(pos, vi);
    }
  }
}

// ---- symmetric 3x3 eigen-decomposition (cyclic Jacobi) --------------------
// Eigenvalues ascending; columns of `vec` are the eigenvectors.
inline void sym_eig3(const Mat3& a_in, Vec3& val, Mat3& vec) {
  Mat3 a = a_in;
  vec = Mat3::identity();
  for (int sweep = 0; sweep < 50; ++sweep) {
    const double off = a(0, 1) * a(0, 1) + a(0, 2) * a(0, 2) + a(1, 2) * a(1, 2);
    const double dg = a(0, 0) * a(0, 0) + a(1, 1) * a(1, 1) + a(2, 2) * a(2, 2);
    if (off <= 1e-36 * dg || off == 0) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        const double apq = a(p, q);
        if (apq == 0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1));
        const double c = 1 / std::sqrt(t * t + 1), s = t * c;
        for (int k = 0; k < 3; ++k) {  // A <- J^T A J
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = vec(k, p), vkq = vec(k, q);
          vec(k, p) = c * vkp - s * vkq;
          vec(k, q) = s * vkp + c * vkq;
        }
      }
  }
  val = Vec3(a(0, 0), a(1, 1), a(2, 2));
  for (int i = 0; i < 2; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (val[j] < val[i]) {
        std::swap(val[i], val[j]);
        const Vec3 ci = vec.col(i), cj = vec.col(j);
        vec.set_col(i, cj); vec.set_col(j, ci);
      }
}

// ---- dense row-major matrix and LDLT with diagonal pivoting ---------------
struct MatX {
  int rows = 0, cols = 0;
  std::vector<double> a;
  MatX() = default;
  MatX(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  double& operator()(int r, int c) { return a[static_cast<size_t>(r) * cols + c]; }
  double operator()(int r, int c) const { return a[static_cast<size_t>(r) * cols + c]; }
};

// Solves M x = b for symmetric M by LDL^T with symmetric diagonal pivoting
// (Eigen::LDLT).  Returns false on a zero pivot or non-finite output.
inline bool ldlt_solve(MatX m, const std::vector<double>& b, std::vector<double>& x) {
  const int n = m.rows;
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  std::vector<double> d(n);
  bool ok = true;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = std::fabs(m(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(m(i, i)) > best) { best = std::fabs(m(i, i)); piv = i; }
    if (piv != k) {
      std::swap(perm[k], perm[piv]);
      for (int c = 0; c < n; ++c) std::swap(m(k, c), m(piv, c));
      for (int r = 0; r < n; ++r) std::swap(m(r, k), m(r, piv));
    }
    // Row k of L from the already-factored columns.
    double dk = m(k, k);
    for (int j = 0; j < k; ++j) dk -= m(k, j) * m(k, j) * d[j];
    d[k] = dk;
    if (!(std::fabs(dk) > DBL_MIN)) { ok = false; d[k] = 0; }
    for (int i = k + 1; i < n; ++i) {
      double s = m(i, k);
      for (int j = 0; j < k; ++j) s -= m(i, j) * m(k, j) * d[j];
      m(i, k) = ok ? s / dk : 0.0;
    }
  }
  if (!ok) return false;
  std::vector<double> y(n);
  for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
  for (int i = 0; i < n; ++i) for (int j = 0; j < i; ++j) y[i] -= m(i, j) * y[j];
  for (int i = 0; i < n; ++i) y[i] /= d[i];
  for (int i = n - 1; i >= 0; --i) for (int j = i + 1; j < n; ++j) y[i] -= m(j, i) * y[j];
  x.assign(n, 0.0);
  for (int i = 0; i < n; ++i) x[perm[i]] = y[i];
  for (double v : x) if (!std::isfinite(v)) return false;
  return true;
}

// Complete-pivoting LU solve of a 4x4 system (Eigen::FullPivLU<Matrix4d>).
inline void fullpiv_lu4_solve(const double a_in[16], const double b[4], double x[4]) {
  double a[4][4];
  for (int r = 0; r < 4; ++r) for (int c = 0; c < 4; ++c) a[r][c] = a_in[r * 4 + c];
  int rp[4] = {0, 1, 2, 3}, cp[4] = {0, 1, 2, 3};
  double rhs[4] = {b[0], b[1], b[2], b[3]};
  for (int k = 0; k < 4; ++k) {
    int pr = k, pc = k;
    double best = -1;
    for (int r = k; r < 4; ++r) for (int c = k; c < 4; ++c)
      if (std::fabs(a[r][c]) > best) { best = std::fabs(a[r][c]); pr = r; pc = c; }
    if (pr != k) { for (int c = 0; c < 4; ++c) std::swap(a[k][c], a[pr][c]); std::swap(rhs[k], rhs[pr]); std::swap(rp[k], rp[pr]); }
    if (pc != k) { for (int r = 0; r < 4; ++r) std::swap(a[r][k], a[r][pc]); std::swap(cp[k], cp[pc]); }
    if (a[k][k] == 0) continue;
    for (int r = k + 1; r < 4; ++r) {
      const double f = a[r][k] / a[k][k];
      a[r][k] = f;
      for (int c = k + 1; c < 4; ++c) a[r][c] -= f * a[k][c];
      rhs[r] -= f * rhs[k];
    }
  }
  double y[4];
  for (int i = 3; i >= 0; --i) {
    double s = rhs[i];
    for (int c = i + 1; c < 4; ++c) s -= a[i][c] * y[c];
    y[i] = a[i][i] != 0 ? s / a[i][i] : 0.0;
  }
  for (int i = 0; i < 4; ++i) x[cp[i]] = y[i];
}

}  // namespace hdo
