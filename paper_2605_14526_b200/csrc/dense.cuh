// Single-CTA dense symmetric LDL^T with Eigen's diagonal pivoting — the
// reference's LDLT<MatrixXd> solves of the contact multiplier system
// (contact.cpp:237-256, Eigen LDLT at :248) and of the reduced adjoint
// multiplier system (backward.cpp:255-262).  Replaces the cuSOLVER potrf/potrs
// pair of round 1: the systems are small (K <= a few hundred rows), so one
// CTA factors them in shared memory inside the PD loop's CUDA graph.
//
// Pivoting.  Eigen's unblocked LDLT (left-looking) picks at step k the
// largest |diagonal| among rows k.. of the ORIGINAL diagonal (the trailing
// diagonal is not updated before its own step), first index on ties, and
// swaps row/column k with it.  The pivot sequence therefore depends only on
// the original diagonal and is computed up front (ldlt_pivots); factoring
// P A P^T without pivoting performs the same arithmetic as the swapping
// algorithm.
//
// Factorization.  Right-looking, one column per step: column j is scaled by
// 1/d_j, then the trailing lower triangle is updated with
// a(i,l) -= (L(i,j) L(l,j)) d_j — per element the same terms in the same
// (ascending j) order as the reference's left-looking sums, so with the same
// input the factors are bitwise the oracle's (explicit round-to-nearest
// products and differences: no FMA contraction).  The triangular solves run
// on one warp (column-oriented forward, then backward substitution).
#pragma once

#include <cfloat>
#include <cuda_runtime.h>

namespace hdk {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// hypot(x, y) bitwise as glibc 2.39's (sysdeps/ieee754/dbl-64/e_hypot.c,
// the non-FMA build: Borges' corrected sqrt(ax^2 + ay^2)), which the
// reference's std::hypot calls (contact.cpp:160-235: slip, tangential
// multiplier norm, cone test).  Checked against the host libm on 2e7 random
// pairs with |args| >= 2^-500; the cone decisions of project_multipliers then
// see the reference's exact values.
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
  double h = __dsqrt_rn(add(mul(ax, ax), mul(ay, ay)));
  double t1, t2;
  if (h <= mul(2.0, ay)) {
    const double delta = sub(h, ay);
    t1 = mul(ax, sub(mul(2.0, delta), ax));
    t2 = mul(sub(delta, mul(2.0, sub(ax, ay))), delta);
  } else {
    const double delta = sub(h, ax);
    t1 = mul(mul(2.0, delta), sub(ax, mul(2.0, ay)));
    t2 = add(mul(sub(mul(4.0, delta), ay), ay), mul(delta, delta));
  }
  return sub(h, __ddiv_rn(add(t1, t2), mul(2.0, h)));
}
__device__ __forceinline__ double libm_hypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) return (isinf(x) || isinf(y)) ? INFINITY : NAN;
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ax > 0x1p+511) {
    if (ay <= mul(ax, 0x1p-54)) return add(ax, ay);
    return __ddiv_rn(hypot_kernel(mul(ax, 0x1p-600), mul(ay, 0x1p-600)), 0x1p-600);
  }
  if (ay < 0x1p-511) {
    if (ax >= __ddiv_rn(ay, 0x1p-54)) return add(ax, ay);
    return mul(hypot_kernel(__ddiv_rn(ax, 0x1p-600), __ddiv_rn(ay, 0x1p-600)), 0x1p-600);
  }
  if (ay <= mul(ax, 0x1p-54)) return add(ax, ay);
  return hypot_kernel(ax, ay);
}

// Pivot order of Eigen's LDLT on the diagonal `diag` (k entries).  perm[s] =
// original index factored at step s.  Scratch: byval, gsz, pos, at (k ints
// each).  Returns (block-uniform) nonzero when a diagonal entry is not finite.
// Elements of equal |diag| form a group; the groups are consumed in
// descending order, and inside a group the members are taken in order of
// their position at the time (a swap moves the element at position s to the
// chosen member's position), which one thread replays.
__device__ int ldlt_pivots(int k, const double* diag, int* perm, int* byval, int* gsz, int* pos, int* at) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double a = fabs(diag[i]);
    if (!isfinite(a)) bad = 1;
    int gt = 0, eq = 0, before = 0;
    for (int j = 0; j < k; ++j) {
      const double b = fabs(diag[j]);
      gt += b > a;
      if (b == a) {
        ++eq;
        before += j < i;
      }
    }
    byval[gt + before] = i;
    gsz[i] = eq;
    pos[i] = i;
    at[i] = i;
  }
  __syncthreads();
  if (bad) return 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < k;) {
      const int m = max(1, gsz[byval[s]]);
      for (int t = 0; t < m; ++t) {
        const int step = s + t;
        int best = -1, bp = 0x7fffffff;
        for (int g = s; g < s + m; ++g) {  // members not yet factored sit at positions >= step
          const int e = byval[g];
          if (pos[e] >= step && pos[e] < bp) {
            bp = pos[e];
            best = e;
          }
        }
        const int displaced = at[step];
        at[bp] = displaced;
        pos[displaced] = bp;
        at[step] = best;
        pos[best] = step;
      }
      s += m;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) perm[i] = at[i];
  __syncthreads();
  return 0;
}

// Lower triangle of a k x k symmetric matrix, packed by columns: column j
// holds rows j..k-1 contiguously (k(k+1)/2 doubles).
struct Packed {
  double* a;
  int n;
  __device__ __forceinline__ size_t col(int j) const { return (size_t)j * n - ((size_t)j * (j - 1)) / 2 - j; }
  __device__ __forceinline__ double& operator()(int i, int j) const { return a[col(j) + i]; }  // i >= j
  static __host__ __device__ size_t doubles(int n) { return (size_t)n * (n + 1) / 2; }
};

// In-place LDL^T of A (already permuted): strict lower <- L, diagonal <- D.
// Returns (block-uniform) nonzero on a pivot with !(|d| > DBL_MIN) or not
// finite (ldlt_solve's failure, la.hpp / Eigen's info()).
__device__ int ldlt_factor(Packed A) {
  __shared__ int bad;
  const int k = A.n;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    double* colj = A.a + A.col(j);
    const double dj = colj[j];
    if (!(fabs(dj) > DBL_MIN) || !isfinite(dj)) {
      if (threadIdx.x == 0) bad = 1;
      break;  // dj is the same value in every thread: uniform exit
    }
    for (int i = j + 1 + threadIdx.x; i < k; i += blockDim.x) colj[i] = colj[i] / dj;
    __syncthreads();
    // trailing update, column l by one warp (round robin), rows i >= l by its lanes
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (int l = j + 1 + warp; l < k; l += nwarps) {
      const double llj = colj[l];
      double* coll = A.a + A.col(l);
      for (int i = l + lane; i < k; i += 32) coll[i] = sub(coll[i], mul(mul(colj[i], llj), dj));
    }
    __syncthreads();
  }
  __syncthreads();
  return bad;
}

// y <- (L D L^T)^{-1} y for the factor of ldlt_factor; warp 0 does the work,
// the whole block must call it.
__device__ void ldlt_substitute(Packed A, double* y) {
  const int k = A.n;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int j = 0; j < k; ++j) {  // L z = y
      const double yj = y[j];
      const double* colj = A.a + A.col(j);
      for (int i = j + 1 + lane; i < k; i += 32) y[i] = sub(y[i], mul(colj[i], yj));
      __syncwarp();
    }
    for (int i = lane; i < k; i += 32) y[i] = y[i] / A(i, i);
    __syncwarp();
    for (int j = k - 1; j > 0; --j) {  // L^T x = z: y_i -= L(j, i) y_j
      const double yj = y[j];
      for (int i = lane; i < j; i += 32) y[i] = sub(y[i], mul(A(j, i), yj));
      __syncwarp();
    }
  }
  __syncthreads();
}

}  // namespace hdk
