// Register-resident fp64 3x3 algebra for the per-element kernels (sm_100a).
//
// One thread owns one tetrahedron; every matrix here lives in registers
// (column-major, vec(F)[3c + r] = F(r, c), the layout of the reference's
// element operator, mesh.hpp:11-14).  The SVD follows the two-sided Jacobi
// sweep of Eigen::JacobiSVD that the reference's signed_svd wraps
// (localstep.cpp:99-114) so U/V sign conventions match it in the generic
// case; the symmetric eigen-solver is a cyclic Jacobi (the reference only
// uses convention-invariant products of its eigenvectors).
#pragma once

#include <cfloat>
#include <cmath>

namespace hdk {

struct M3 {
  double m[9];
  __device__ __forceinline__ double& operator()(int r, int c) { return m[r + 3 * c]; }
  __device__ __forceinline__ double operator()(int r, int c) const { return m[r + 3 * c]; }
};
struct V3 {
  double v[3];
  __device__ __forceinline__ double& operator[](int i) { return v[i]; }
  __device__ __forceinline__ double operator[](int i) const { return v[i]; }
};

__device__ __forceinline__ V3 v3(double a, double b, double c) { V3 r; r.v[0] = a; r.v[1] = b; r.v[2] = c; return r; }
__device__ __forceinline__ M3 m3_identity() {
  M3 a;
#pragma unroll
  for (int i = 0; i < 9; ++i) a.m[i] = 0.0;
  a.m[0] = a.m[4] = a.m[8] = 1.0;
  return a;
}
__device__ __forceinline__ M3 m3_zero() {
  M3 a;
#pragma unroll
  for (int i = 0; i < 9; ++i) a.m[i] = 0.0;
  return a;
}
__device__ __forceinline__ M3 mul(const M3& a, const M3& b) {
  M3 o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o(r, c) = a(r, 0) * b(0, c) + a(r, 1) * b(1, c) + a(r, 2) * b(2, c);
  return o;
}
// a^T b
__device__ __forceinline__ M3 mul_tn(const M3& a, const M3& b) {
  M3 o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o(r, c) = a(0, r) * b(0, c) + a(1, r) * b(1, c) + a(2, r) * b(2, c);
  return o;
}
// a b^T
__device__ __forceinline__ M3 mul_nt(const M3& a, const M3& b) {
  M3 o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o(r, c) = a(r, 0) * b(c, 0) + a(r, 1) * b(c, 1) + a(r, 2) * b(c, 2);
  return o;
}
// u diag(s) v^T
__device__ __forceinline__ M3 recompose(const M3& u, const V3& s, const M3& v) {
  M3 o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o(r, c) = u(r, 0) * s[0] * v(c, 0) + u(r, 1) * s[1] * v(c, 1) + u(r, 2) * s[2] * v(c, 2);
  return o;
}
__device__ __forceinline__ double det3(const M3& a) {
  return a(0, 0) * (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) - a(1, 0) * (a(0, 1) * a(2, 2) - a(0, 2) * a(2, 1)) +
         a(2, 0) * (a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1));
}
__device__ __forceinline__ double dot3(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
__device__ __forceinline__ double norm3(const V3& a) { return sqrt(dot3(a, a)); }

// ---- Eigen::JacobiSVD<Matrix3d> sweep --------------------------------------
struct Rot { double c, s; };
__device__ __forceinline__ void rows_rot(M3& m, int p, int q, double c, double s) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double x = m(p, i), y = m(q, i);
    m(p, i) = c * x + s * y;
    m(q, i) = -s * x + c * y;
  }
}
// applyOnTheRight(p, q, (c, s)): columns rotated by the transpose.
__device__ __forceinline__ void cols_rot(M3& m, int p, int q, double c, double s) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double x = m(i, p), y = m(i, q);
    m(i, p) = c * x - s * y;
    m(i, q) = s * x + c * y;
  }
}
__device__ __forceinline__ void svd_pair(M3& w, M3& u, M3& v, int p, int q, double& max_diag) {
  const double m00 = w(p, p), m01 = w(p, q), m10 = w(q, p), m11 = w(q, q);
  double c1 = 1.0, s1 = 0.0;
  const double t = m00 + m11, d = m10 - m01;
  if (fabs(d) >= DBL_MIN) {
    const double uu = t / d;
    const double tmp = sqrt(1.0 + uu * uu);
    s1 = 1.0 / tmp;
    c1 = uu / tmp;
  }
  const double n00 = c1 * m00 + s1 * m10, n01 = c1 * m01 + s1 * m11, n11 = -s1 * m01 + c1 * m11;
  double cr = 1.0, sr = 0.0;
  const double deno = 2.0 * fabs(n01);
  if (deno >= DBL_MIN) {
    const double tau = (n00 - n11) / deno;
    const double w2 = sqrt(tau * tau + 1.0);
    const double tt = tau > 0 ? 1.0 / (tau + w2) : 1.0 / (tau - w2);
    const double sgn = tt > 0 ? 1.0 : -1.0;
    const double n = 1.0 / sqrt(tt * tt + 1.0);
    sr = -sgn * copysign(1.0, n01) * fabs(tt) * n;  // n01 / |n01|, exactly
    cr = n;
  }
  // j_left = rot1 * j_right^T
  const double cl = c1 * cr + s1 * sr, sl = -c1 * sr + s1 * cr;
  rows_rot(w, p, q, cl, sl);
  cols_rot(u, p, q, cl, -sl);
  cols_rot(w, p, q, cr, sr);
  cols_rot(v, p, q, cr, sr);
  max_diag = fmax(max_diag, fmax(fabs(w(p, p)), fabs(w(q, q))));
}

// Rotation-normalised SVD (signed_svd, localstep.cpp:99-114): det U = det V = +1,
// a reflection folds into sigma[2].
__device__ __forceinline__ void signed_svd(const M3& f, M3& u, V3& sig, M3& v) {
  double scale = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) scale = fmax(scale, fabs(f.m[i]));
  if (scale == 0.0) scale = 1.0;
  M3 w;
#pragma unroll
  for (int i = 0; i < 9; ++i) w.m[i] = f.m[i] / scale;
  u = m3_identity();
  v = m3_identity();
  const double precision = 2.0 * DBL_EPSILON;
  double max_diag = fmax(fabs(w(0, 0)), fmax(fabs(w(1, 1)), fabs(w(2, 2))));
  for (int sweep = 0; sweep < 64; ++sweep) {
    bool finished = true;
    // pairs (p, q) = (1,0), (2,0), (2,1) in Eigen's loop order
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int p = k == 0 ? 1 : 2, q = k == 2 ? 1 : 0;
      const double thr = fmax(DBL_MIN, precision * max_diag);
      if (fabs(w(p, q)) > thr || fabs(w(q, p)) > thr) {
        finished = false;
        svd_pair(w, u, v, p, q, max_diag);
      }
    }
    if (finished) break;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double d = w(i, i);
    sig[i] = fabs(d) * scale;
    if (d < 0) { u(0, i) = -u(0, i); u(1, i) = -u(1, i); u(2, i) = -u(2, i); }
  }
  // descending sort with Eigen's first-max swaps (swap partners are compile-
  // time indices, so sig, u and v stay in registers)
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    int pos = i;
    double best = sig[i];
#pragma unroll
    for (int k = i + 1; k < 3; ++k)
      if (sig[k] > best) { best = sig[k]; pos = k; }
#pragma unroll
    for (int k = i + 1; k < 3; ++k)
      if (pos == k) {
        const double ts = sig[i]; sig[i] = sig[k]; sig[k] = ts;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          double t = u(r, i); u(r, i) = u(r, k); u(r, k) = t;
          t = v(r, i); v(r, i) = v(r, k); v(r, k) = t;
        }
      }
  }
  if (det3(u) < 0) { u(0, 2) = -u(0, 2); u(1, 2) = -u(1, 2); u(2, 2) = -u(2, 2); sig[2] = -sig[2]; }
  if (det3(v) < 0) { v(0, 2) = -v(0, 2); v(1, 2) = -v(1, 2); v(2, 2) = -v(2, 2); sig[2] = -sig[2]; }
}

// Cyclic-Jacobi eigen-decomposition of a symmetric 3x3; ascending values.
__device__ __forceinline__ void sym_eig(const M3& a_in, V3& val, M3& vec) {
  M3 a = a_in;
  vec = m3_identity();
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = a(0, 1) * a(0, 1) + a(0, 2) * a(0, 2) + a(1, 2) * a(1, 2);
    const double dg = a(0, 0) * a(0, 0) + a(1, 1) * a(1, 1) + a(2, 2) * a(2, 2);
    if (off <= 1e-36 * dg || off == 0.0) break;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int p = k == 2 ? 1 : 0, q = k == 0 ? 1 : 2;
      const double apq = a(p, q);
      if (apq == 0.0) continue;
      const double theta = (a(q, q) - a(p, p)) / (2.0 * apq);
      const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double x = a(i, p), y = a(i, q);
        a(i, p) = c * x - s * y;
        a(i, q) = s * x + c * y;
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double x = a(p, i), y = a(q, i);
        a(p, i) = c * x - s * y;
        a(q, i) = s * x + c * y;
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double x = vec(i, p), y = vec(i, q);
        vec(i, p) = c * x - s * y;
        vec(i, q) = s * x + c * y;
      }
    }
  }
  val = v3(a(0, 0), a(1, 1), a(2, 2));
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = i + 1; j < 3; ++j)
      if (val[j] < val[i]) {
        const double t = val[i]; val[i] = val[j]; val[j] = t;
#pragma unroll
        for (int r = 0; r < 3; ++r) { const double x = vec(r, i); vec(r, i) = vec(r, j); vec(r, j) = x; }
      }
}

// V diag(d) V^T
__device__ __forceinline__ M3 eig_recompose(const M3& vec, const V3& d) { return recompose(vec, d, vec); }

// ---- stretch-space densities (localstep.cpp:116-174) -------------------------
struct StretchNH {
  double mu, lambda;
  __device__ __forceinline__ double value(const V3& s) const {
    const double L = log(s[0] * s[1] * s[2]);
    return 0.5 * mu * (s[0] * s[0] + s[1] * s[1] + s[2] * s[2] - 3.0) - mu * L + 0.5 * lambda * L * L;
  }
  __device__ __forceinline__ V3 gradient(const V3& s) const {
    const double L = log(s[0] * s[1] * s[2]);
    V3 g;
#pragma unroll
    for (int i = 0; i < 3; ++i) g[i] = mu * (s[i] - 1.0 / s[i]) + lambda * L / s[i];
    return g;
  }
  __device__ __forceinline__ M3 hessian(const V3& s) const {
    const double L = log(s[0] * s[1] * s[2]);
    M3 h;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (i == j) {
          const double inv2 = 1.0 / (s[i] * s[i]);
          h(i, i) = mu * (1.0 + inv2) + lambda * (1.0 - L) * inv2;
        } else {
          h(i, j) = lambda / (s[i] * s[j]);
        }
      }
    return h;
  }
  // The same Hessian as diag(d) + lambda u u^T, u_i = 1 / s_i.
  __device__ __forceinline__ void diag_rank1(const V3& s, V3& d, V3& u) const {
    const double L = log(s[0] * s[1] * s[2]);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      u[i] = 1.0 / s[i];
      d[i] = mu * (1.0 + u[i] * u[i]) - lambda * L * (u[i] * u[i]);
    }
  }
};
struct StretchBarrier {
  double mu, lambda;
  __device__ __forceinline__ double value(const V3& s) const {
    const double L = log(s[0] * s[1] * s[2]);
    return -mu * L + 0.5 * lambda * L * L;
  }
  __device__ __forceinline__ V3 gradient(const V3& s) const {
    const double L = log(s[0] * s[1] * s[2]);
    V3 g;
#pragma unroll
    for (int i = 0; i < 3; ++i) g[i] = (-mu + lambda * L) / s[i];
    return g;
  }
  __device__ __forceinline__ M3 hessian(const V3& s) const {
    const double L = log(s[0] * s[1] * s[2]);
    M3 h;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (i == j) h(i, i) = (mu - lambda * (L - 1.0)) / (s[i] * s[i]);
        else h(i, j) = lambda / (s[i] * s[j]);
      }
    return h;
  }
  __device__ __forceinline__ void diag_rank1(const V3& s, V3& d, V3& u) const {
    const double L = log(s[0] * s[1] * s[2]);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      u[i] = 1.0 / s[i];
      d[i] = (mu - lambda * L) * (u[i] * u[i]);
    }
  }
};

constexpr double kSigmaFloor = 1e-6;
constexpr int kNewtonCap = 50;
constexpr int kBacktrackCap = 30;

__device__ __forceinline__ V3 vmax_floor(const V3& s) { return v3(fmax(s[0], kSigmaFloor), fmax(s[1], kSigmaFloor), fmax(s[2], kSigmaFloor)); }

// Safeguarded Newton on the principal stretches (newton_on_stretches,
// localstep.cpp:35-83).  Returns false when stationarity is not reached
// (ProxDiverged).
// 1: always take the eigen path (A/B of the Sherman-Morrison direction; set by
// hdk_set_newton_eigen from HETERODYN_NEWTON_EIGEN).
__device__ int g_newton_eigen = 0;

// The accepted candidate's gradient, residual norm and objective are those
// of the next iterate, so they carry over instead of being re-evaluated
// (same expressions on the same values: bitwise the re-evaluated ones; the
// log and six divisions of a gradient dominate an iteration).
template <class D>
__device__ __forceinline__ bool newton_stretch(const V3& sf, double k, const D& den, V3& s_out, int& iters) {
  V3 s = vmax_floor(sf);
  const double tol = 1e-10 * k;
  V3 r;
  double r0, f0;
  {
    const V3 g = den.gradient(s);
    r = v3(k * (s[0] - sf[0]) + g[0], k * (s[1] - sf[1]) + g[1], k * (s[2] - sf[2]) + g[2]);
    r0 = norm3(r);
    const V3 d0 = v3(s[0] - sf[0], s[1] - sf[1], s[2] - sf[2]);
    f0 = 0.5 * k * dot3(d0, d0) + den.value(s);
  }
  int it = 0;
  for (; it < kNewtonCap; ++it) {
    if (r0 <= tol) break;
    const double lo = 1e-8 * k;
    V3 dir;
    // H + k I = diag(D) + lambda u u^T.  With lambda >= 0 its eigenvalues are
    // at least min D (interlacing), so when min D >= the floor 1e-8 k the
    // floored eigen-solve of localstep.cpp:57-66 is the plain inverse:
    // Sherman-Morrison, no 3x3 eigen-decomposition.  Otherwise the floor can
    // act and the eigen path runs as in the reference.
    V3 dd, u;
    den.diag_rank1(s, dd, u);
    const double D0 = dd[0] + k, D1 = dd[1] + k, D2 = dd[2] + k;
    if (!g_newton_eigen && den.lambda >= 0.0 && fmin(D0, fmin(D1, D2)) >= lo) {
      const V3 a = v3(r[0] / D0, r[1] / D1, r[2] / D2), b = v3(u[0] / D0, u[1] / D1, u[2] / D2);
      const double c = den.lambda * dot3(u, a) / (1.0 + den.lambda * dot3(u, b));
#pragma unroll
      for (int i = 0; i < 3; ++i) dir[i] = -(a[i] - b[i] * c);
    } else {
      M3 h = den.hessian(s);
      h(0, 0) += k; h(1, 1) += k; h(2, 2) += k;
      V3 lam;
      M3 ev;
      sym_eig(h, lam, ev);
      V3 pr;
#pragma unroll
      for (int i = 0; i < 3; ++i) pr[i] = (ev(0, i) * r[0] + ev(1, i) * r[1] + ev(2, i) * r[2]) / fmax(lam[i], lo);
#pragma unroll
      for (int i = 0; i < 3; ++i) dir[i] = -(ev(i, 0) * pr[0] + ev(i, 1) * pr[1] + ev(i, 2) * pr[2]);
    }
    const double slope = dot3(r, dir);
    double t = 1.0;
    bool accepted = false;
    for (int bt = 0; bt < kBacktrackCap; ++bt, t *= 0.5) {
      const V3 cand = vmax_floor(v3(s[0] + t * dir[0], s[1] + t * dir[1], s[2] + t * dir[2]));
      const V3 dc = v3(cand[0] - sf[0], cand[1] - sf[1], cand[2] - sf[2]);
      const double fc = 0.5 * k * dot3(dc, dc) + den.value(cand);
      const bool obj_ok = fc <= f0 + 1e-4 * t * slope;
      const V3 gc = den.gradient(cand);
      const V3 rc = v3(k * dc[0] + gc[0], k * dc[1] + gc[1], k * dc[2] + gc[2]);
      const double nc = norm3(rc);
      const bool res_ok = nc <= (1.0 - 1e-4 * t) * r0;
      if (obj_ok || res_ok) {
        s = cand;
        r = rc;
        r0 = nc;
        f0 = fc;
        accepted = true;
        break;
      }
    }
    if (!accepted) break;
  }
  s_out = s;
  iters = it;
  return r0 <= tol;
}

// Complete-pivoting 4x4 solve (FullPivLU, localstep.cpp:215,395); a is
// row-major and destroyed.
__device__ __forceinline__ void lu4_solve(double a[16], double rhs[4], double x[4]) {
  int cp[4] = {0, 1, 2, 3};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int pr = k, pc = k;
    double best = -1.0;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (r >= k && c >= k && fabs(a[r * 4 + c]) > best) { best = fabs(a[r * 4 + c]); pr = r; pc = c; }
    if (pr != k) {
#pragma unroll
      for (int c = 0; c < 4; ++c) { const double t = a[k * 4 + c]; a[k * 4 + c] = a[pr * 4 + c]; a[pr * 4 + c] = t; }
      const double t = rhs[k]; rhs[k] = rhs[pr]; rhs[pr] = t;
    }
    if (pc != k) {
#pragma unroll
      for (int r = 0; r < 4; ++r) { const double t = a[r * 4 + k]; a[r * 4 + k] = a[r * 4 + pc]; a[r * 4 + pc] = t; }
      const int t = cp[k]; cp[k] = cp[pc]; cp[pc] = t;
    }
    const double piv = a[k * 4 + k];
    if (piv != 0.0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (r <= k) continue;
        const double f = a[r * 4 + k] / piv;
        a[r * 4 + k] = f;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c > k) a[r * 4 + c] -= f * a[k * 4 + c];
        rhs[r] -= f * rhs[k];
      }
    }
  }
  double y[4];
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    double s = rhs[i];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c > i) s -= a[i * 4 + c] * y[c];
    y[i] = a[i * 4 + i] != 0.0 ? s / a[i * 4 + i] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (cp[i] == j) x[j] = y[i];
  }
}

// Unit-volume projection in stretch space (volume_project, localstep.cpp:181-237).
__device__ __forceinline__ bool volume_stretch(const V3& sf, V3& s_out) {
  const V3 cl = vmax_floor(sf);
  const double scale = pow(cl[0] * cl[1] * cl[2], -1.0 / 3.0);
  V3 s = v3(cl[0] * scale, cl[1] * scale, cl[2] * scale);
  double gamma = 0.0;
  const double tol = 1e-10 * fmax(1.0, fmax(fabs(sf[0]), fmax(fabs(sf[1]), fabs(sf[2]))));
  auto residual = [&](const V3& x, double g, double out[4]) {
    const double jx = x[0] * x[1] * x[2];
#pragma unroll
    for (int i = 0; i < 3; ++i) out[i] = x[i] - sf[i] + g * jx / x[i];
    out[3] = jx - 1.0;
  };
  for (int it = 0; it < kNewtonCap; ++it) {
    double res[4];
    residual(s, gamma, res);
    const double m0 = res[0] * res[0] + res[1] * res[1] + res[2] * res[2] + res[3] * res[3];
    if (sqrt(m0) <= tol) break;
    const double jx = s[0] * s[1] * s[2];
    double kkt[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) kkt[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      kkt[i * 4 + i] = 1.0;
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (i != j) kkt[i * 4 + j] = gamma * jx / (s[i] * s[j]);
      kkt[i * 4 + 3] = jx / s[i];
      kkt[12 + i] = jx / s[i];
    }
    double rhs[4] = {-res[0], -res[1], -res[2], -res[3]}, step[4];
    lu4_solve(kkt, rhs, step);
    double t = 1.0;
    bool accepted = false;
    for (int bt = 0; bt < kBacktrackCap; ++bt, t *= 0.5) {
      const V3 cand = vmax_floor(v3(s[0] + t * step[0], s[1] + t * step[1], s[2] + t * step[2]));
      const double cg = gamma + t * step[3];
      double rc[4];
      residual(cand, cg, rc);
      if (rc[0] * rc[0] + rc[1] * rc[1] + rc[2] * rc[2] + rc[3] * rc[3] < m0 * (1.0 - 1e-4 * t)) {
        s = cand;
        gamma = cg;
        accepted = true;
        break;
      }
    }
    if (!accepted) break;
  }
  double res[4];
  residual(s, gamma, res);
  s_out = s;
  return sqrt(res[0] * res[0] + res[1] * res[1] + res[2] * res[2] + res[3] * res[3]) <= tol;
}

// Hat-space pair coefficients of the prox differential
// (ProxDifferential::ProxDifferential, localstep.cpp:305-336).
__device__ __forceinline__ void pair_coefficients(const V3& sf, const V3& mapped, double pa[3], double pb[3]) {
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const int i = p == 2 ? 1 : 0, j = p == 0 ? 1 : 2;
    const double si = sf[i], sj = sf[j];
    double d2 = sj * sj - si * si;
    const double f2 = 1e-10 * fmax(1.0, fmax(si * si, sj * sj));
    if (fabs(d2) < f2) d2 = d2 >= 0 ? f2 : -f2;
    const double cu = (mapped[j] - mapped[i]) * (sj + si) / d2;
    double ds = si + sj;
    const double f1 = 1e-10 * fmax(1.0, fmax(fabs(si), fabs(sj)));
    if (fabs(ds) < f1) ds = ds >= 0 ? f1 : -f1;
    const double cw = (mapped[i] + mapped[j]) / ds;
    pa[p] = 0.5 * (cu + cw);
    pb[p] = 0.5 * (cu - cw);
  }
}

}  // namespace hdk
