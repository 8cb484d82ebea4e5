// Preconditioned conjugate gradients for the adjoint backbone (the B200
// alternative to the reference's Anderson fixed point, backward.cpp:170-204):
// the backbone solves (A - B) x = s, and the reference iterates
// x <- A^{-1}(s + B x) with AA(8) until ||t - x|| <= 1e-10 ||t||,
// t = A^{-1}(s + B x).  Since t - x = A^{-1}(s - (A - B) x) = A^{-1} r is the
// A^{-1}-preconditioned residual z of CG on the same system, CG with the
// same preconditioner stops on exactly the reference's test and returns
// x + z (the reference's t).  A - B is symmetric (backward.cpp:117-163);
// where it is not positive definite along a search direction (p.q <= 0) the
// iteration reports it and the engine falls back to the Anderson backbone.
//
// Vectors are in elimination order [n][3] (the solve's layout); reductions
// are fixed-grid partials folded by the last block (ticket), so results are
// bitwise reproducible.
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/hdk.h"
#include "launch.cuh"

namespace {

constexpr int kT = 256;
constexpr int kB = HDK_RED_BLOCKS;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block partial sums of NQ quantities into partial[q * kB + block].
template <int NQ>
__device__ __forceinline__ void block_store(const double (&v)[NQ], double* partial) {
  __shared__ double sm[kT / 32][NQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double s = warp_sum(v[q]);
    if (lane == 0) sm[warp][q] = s;
  }
  __syncthreads();
  if (threadIdx.x < NQ) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) s += sm[w][threadIdx.x];
    partial[threadIdx.x * kB + blockIdx.x] = s;
  }
}

// True in the block that finishes last (its loads of the others' partials
// are ordered after their stores).
__device__ __forceinline__ bool last_block(unsigned int* ticket) {
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(ticket, 1u);
    is_last = t == gridDim.x - 1;
    if (is_last) *ticket = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last != 0;
}

// Fixed-order fold of partial quantity q over the kB blocks (one warp).
__device__ __forceinline__ double fold(const double* partial, int q) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int b = lane; b < kB; b += 32) s += partial[q * kB + b];
  return warp_sum(s);
}

// r = s - A x0 + R(x0) (R = gather o B): the residual of x0 = A^{-1} s.
__global__ void k_pcg_r0(int n3, const double* __restrict__ s, const double* __restrict__ ax,
                         const double* __restrict__ rx, double* __restrict__ r) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n3) r[i] = (s[i] - ax[i]) + rx[i];
}

// y = A p on the three axes (A_ff in elimination order, columns are positions).
__global__ void k_pcg_spmv(hdk_csr A, const double* __restrict__ p, double* __restrict__ y, const hdk_pcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (st->cond == 0) return;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.rows) return;
  double y0 = 0.0, y1 = 0.0, y2 = 0.0;
  for (int k = A.off[row]; k < A.off[row + 1]; ++k) {
    const double w = A.val[k];
    const double* v = p + 3 * (size_t)A.col[k];
    y0 += w * v[0];
    y1 += w * v[1];
    y2 += w * v[2];
  }
  y[3 * (size_t)row] = y0;
  y[3 * (size_t)row + 1] = y1;
  y[3 * (size_t)row + 2] = y2;
}

// After z = A^{-1} r: rz = r.z, the reference's convergence test on
// (x, z), beta, and the WHILE condition.
__global__ void __launch_bounds__(kT) k_pcg_rz(int n3, const double* __restrict__ r, const double* __restrict__ z,
                                               const double* __restrict__ x, double* partial, unsigned int* ticket,
                                               hdk_pcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (st->cond == 0) return;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int i = blockIdx.x * kT + threadIdx.x; i < n3; i += kB * kT) {
    const double zi = z[i], t = x[i] + zi;
    acc[0] += r[i] * zi;
    acc[1] += zi * zi;
    acc[2] += t * t;
  }
  block_store<3>(acc, partial);
  if (!last_block(ticket)) return;
  if (threadIdx.x >= 32) return;
  const double rz = fold(partial, 0), zz = fold(partial, 1), tt = fold(partial, 2);
  if (threadIdx.x != 0) return;
  const int it = st->iter + 1;  // solves so far
  st->iter = it;
  const bool done = sqrt(zz) <= st->tol * fmax(sqrt(tt), 1e-30);
  st->beta = st->rz > 0.0 && it > 1 ? rz / st->rz : 0.0;
  st->rz = rz;
  st->done = done ? 1 : 0;
  if (!done && it >= st->k_max) st->err = 10;  // AdjointDiverged (cap)
  if (!isfinite(rz)) st->err = 10;
  st->cond = (!done && st->err == 0) ? 1 : 0;
}

// The WHILE condition from the state (last kernel of the loop body; any
// kernel above may have ended the loop).
__global__ void k_pcg_cond(const hdk_pcg* st, cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (use_handle) cudaGraphSetConditional(handle, st->cond);
}

// p = z + beta p, and p by vertex (the B apply's input; fixed vertices stay 0).
__global__ void k_pcg_p(int n, const double* __restrict__ z, double* __restrict__ p, double* __restrict__ pv,
                        const int* __restrict__ p2v, const hdk_pcg* st, cudaGraphConditionalHandle handle,
                        int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  // the loop body's last kernel: the WHILE condition is final here
  if (use_handle && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(handle, st->cond);
  if (st->cond == 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * n) return;
  const double b = st->beta;
  const double v = z[i] + b * p[i];
  p[i] = v;
  const int row = i / 3;
  pv[3 * (size_t)__ldg(p2v + row) + (i - 3 * row)] = v;
}

// q = A p - R(p), p.q, alpha = rz / p.q (last block); p.q <= 0 ends the loop
// with err = -1 (the engine falls back to the Anderson backbone).
__global__ void __launch_bounds__(kT) k_pcg_q(int n3, const double* __restrict__ ap, const double* __restrict__ rp,
                                              const double* __restrict__ p, double* __restrict__ q, double* partial,
                                              unsigned int* ticket, hdk_pcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (st->cond == 0) return;
  double acc[1] = {0.0};
  for (int i = blockIdx.x * kT + threadIdx.x; i < n3; i += kB * kT) {
    const double qi = ap[i] - rp[i];
    q[i] = qi;
    acc[0] += p[i] * qi;
  }
  block_store<1>(acc, partial);
  if (!last_block(ticket)) return;
  if (threadIdx.x >= 32) return;
  const double pq = fold(partial, 0);
  if (threadIdx.x != 0) return;
  st->pq = pq;
  if (!(pq > 0.0)) {
    st->err = -1;
    st->cond = 0;
  } else {
    st->alpha = st->rz / pq;
  }
}

// Fused: R(p) = gather o B p from the sorted element forces (8 lanes per row,
// the gather's lane split and fold), A p (A_ff row, 8 lanes), q = A p - R(p),
// p.q and alpha = rz / p.q (last block).
__global__ void __launch_bounds__(kT) k_pcg_apply(hdk_vtx x, hdk_csr A, const double* __restrict__ ef,
                                                  const double* __restrict__ p, double* __restrict__ q, double* partial,
                                                  unsigned int* ticket, hdk_pcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (st->cond == 0) return;
  const int sub = threadIdx.x & 7, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[1] = {0.0};
  // a warp takes four consecutive rows per round (warp-uniform loop: the
  // shuffle folds below need every lane)
  for (int rb = blockIdx.x * (kT / 8) + 4 * warp; rb < x.n; rb += kB * (kT / 8)) {
    const int row = rb + (lane >> 3);
    const bool live = row < x.n;
    double r0 = 0.0, r1 = 0.0, r2 = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const int e = live ? __ldg(x.pinc_off + row + 1) : 0;
    for (int j = (live ? __ldg(x.pinc_off + row) : 0) + sub; j < e; j += 8) {
      const double* f = ef + 3 * (size_t)j;
      r0 += __ldg(f);
      r1 += __ldg(f + 1);
      r2 += __ldg(f + 2);
    }
    const int ke = live ? __ldg(A.off + row + 1) : 0;
    for (int k = (live ? __ldg(A.off + row) : 0) + sub; k < ke; k += 8) {
      const double w = __ldg(A.val + k);
      const double* v = p + 3 * (size_t)__ldg(A.col + k);
      a0 += w * v[0];
      a1 += w * v[1];
      a2 += w * v[2];
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      r0 += __shfl_xor_sync(0xffffffffu, r0, o);
      r1 += __shfl_xor_sync(0xffffffffu, r1, o);
      r2 += __shfl_xor_sync(0xffffffffu, r2, o);
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (sub == 0 && live) {
      const double q0 = a0 - r0, q1 = a1 - r1, q2 = a2 - r2;
      double* qr = q + 3 * (size_t)row;
      qr[0] = q0;
      qr[1] = q1;
      qr[2] = q2;
      const double* pr = p + 3 * (size_t)row;
      acc[0] += (pr[0] * q0 + pr[1] * q1) + pr[2] * q2;
    }
  }
  block_store<1>(acc, partial);
  if (!last_block(ticket)) return;
  if (threadIdx.x >= 32) return;
  const double pq = fold(partial, 0);
  if (threadIdx.x != 0) return;
  st->pq = pq;
  if (!(pq > 0.0)) {
    st->err = -1;
    st->cond = 0;
  } else {
    st->alpha = st->rz / pq;
  }
}

// x += alpha p, r -= alpha q.
__global__ void k_pcg_xr(int n3, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                         const double* __restrict__ q, const hdk_pcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (st->cond == 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const double a = st->alpha;
  x[i] += a * p[i];
  r[i] -= a * q[i];
}

// x_full = x + z by vertex (the reference returns t = x + A^{-1} r).
__global__ void k_pcg_final(int n, const double* __restrict__ x, const double* __restrict__ z, double* __restrict__ xv,
                            const int* __restrict__ p2v) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * n) return;
  const int row = i / 3;
  xv[3 * (size_t)__ldg(p2v + row) + (i - 3 * row)] = x[i] + z[i];
}

__global__ void k_pcg_init(hdk_pcg* st, double tol, int k_max) {
  st->rz = st->pq = st->alpha = st->beta = 0.0;
  st->tol = tol;
  st->iter = 0;
  st->k_max = k_max;
  st->done = 0;
  st->err = 0;
  st->cond = 1;
}

inline int nb(long long n) { return static_cast<int>((n + 255) / 256 > 0 ? (n + 255) / 256 : 1); }
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
inline int last() { return static_cast<int>(cudaGetLastError()); }

}  // namespace

extern "C" {

HDK_API int hdk_pcg_init(hdk_pcg* st, double tol, int k_max, void* stream) {
  hdk::launch(k_pcg_init, dim3(1), dim3(1), 0, S(stream), st, tol, k_max);
  return last();
}
HDK_API int hdk_pcg_r0(int n3, const double* s, const double* ax, const double* rx, double* r, void* stream) {
  hdk::launch(k_pcg_r0, dim3(nb(n3)), dim3(256), 0, S(stream), n3, s, ax, rx, r);
  return last();
}
HDK_API int hdk_pcg_spmv(const hdk_csr* a, const double* p, double* y, const hdk_pcg* st, void* stream) {
  hdk::launch(k_pcg_spmv, dim3(nb(a->rows)), dim3(256), 0, S(stream), *a, p, y, st);
  return last();
}
HDK_API int hdk_pcg_rz(int n3, const double* r, const double* z, const double* x, double* partial,
                       unsigned int* ticket, hdk_pcg* st, void* stream) {
  hdk::launch(k_pcg_rz, dim3(kB), dim3(kT), 0, S(stream), n3, r, z, x, partial, ticket, st);
  return last();
}
HDK_API int hdk_pcg_cond(const hdk_pcg* st, unsigned long long cond_handle, void* stream) {
  hdk::launch(k_pcg_cond, dim3(1), dim3(1), 0, S(stream), st, static_cast<cudaGraphConditionalHandle>(cond_handle),
              cond_handle ? 1 : 0);
  return last();
}
HDK_API int hdk_pcg_p(int n, const double* z, double* p, double* pv, const int* p2v, const hdk_pcg* st,
                      unsigned long long cond_handle, void* stream) {
  hdk::launch(k_pcg_p, dim3(nb(3LL * n)), dim3(256), 0, S(stream), n, z, p, pv, p2v, st,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle ? 1 : 0);
  return last();
}
HDK_API int hdk_pcg_apply(const hdk_vtx* x, const hdk_csr* a, const double* ef_sorted, const double* p, double* q,
                          double* partial, unsigned int* ticket, hdk_pcg* st, void* stream) {
  if (!x->pinc_off) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_pcg_apply, dim3(kB), dim3(kT), 0, S(stream), *x, *a, ef_sorted, p, q, partial, ticket, st);
  return last();
}
HDK_API int hdk_pcg_q(int n3, const double* ap, const double* rp, const double* p, double* q, double* partial,
                      unsigned int* ticket, hdk_pcg* st, void* stream) {
  hdk::launch(k_pcg_q, dim3(kB), dim3(kT), 0, S(stream), n3, ap, rp, p, q, partial, ticket, st);
  return last();
}
HDK_API int hdk_pcg_xr(int n3, double* x, double* r, const double* p, const double* q, const hdk_pcg* st,
                       void* stream) {
  hdk::launch(k_pcg_xr, dim3(nb(n3)), dim3(256), 0, S(stream), n3, x, r, p, q, st);
  return last();
}
HDK_API int hdk_pcg_final(int n, const double* x, const double* z, double* x_full, const int* p2v, void* stream) {
  hdk::launch(k_pcg_final, dim3(nb(3LL * n)), dim3(256), 0, S(stream), n, x, z, x_full, p2v);
  return last();
}

}  // extern "C"

// ---- segmented batch (lockstep engine): one CG per sample ---------------------
// Sample s owns elimination rows [s n, (s+1) n); its reductions run on blockIdx.y
// = s with their own partials (stride HDK_SEG_PSTRIDE) and ticket; every kernel
// skips a sample whose loop has ended.  *any (the solve's run flag and the WHILE
// condition) is the OR over the samples.
namespace {

// blocks per sample of the per-sample CG kernels (<= 32: one lane per block
// partial in fold_rb): twice the other segmented kernels' HDK_SEG_RB, so a
// C5 sample's 5,950 rows take ~6 passes per thread instead of ~12
constexpr int kSRB = 2 * HDK_SEG_RB;
static_assert(kSRB <= 32, "fold_rb folds one partial per lane");

template <int NQ>
__device__ __forceinline__ void block_store_rb(const double (&v)[NQ], double* partial) {
  __shared__ double sm[kT / 32][NQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double s = warp_sum(v[q]);
    if (lane == 0) sm[warp][q] = s;
  }
  __syncthreads();
  if (threadIdx.x < NQ) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) s += sm[w][threadIdx.x];
    partial[threadIdx.x * kSRB + blockIdx.x] = s;
  }
}
__device__ __forceinline__ double fold_rb(const double* partial, int q) {
  const int lane = threadIdx.x & 31;
  const double v = lane < kSRB ? partial[q * kSRB + lane] : 0.0;
  return warp_sum(v);
}

__global__ void k_spcg_init(hdk_pcg* st, int count, double tol, int k_max, int* any) {
  for (int s = threadIdx.x; s < count; s += blockDim.x) {
    hdk_pcg* c = st + s;
    c->rz = c->pq = c->alpha = c->beta = 0.0;
    c->tol = tol;
    c->iter = 0;
    c->k_max = k_max;
    c->done = 0;
    c->err = 0;
    c->cond = 1;
  }
  if (threadIdx.x == 0) *any = 1;
}

__global__ void k_spcg_spmv(hdk_csr A, int ns, const double* __restrict__ p, double* __restrict__ y,
                            const hdk_pcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.rows || st[row / ns].cond == 0) return;
  double y0 = 0.0, y1 = 0.0, y2 = 0.0;
  for (int k = A.off[row]; k < A.off[row + 1]; ++k) {
    const double w = A.val[k];
    const double* v = p + 3 * (size_t)A.col[k];
    y0 += w * v[0];
    y1 += w * v[1];
    y2 += w * v[2];
  }
  y[3 * (size_t)row] = y0;
  y[3 * (size_t)row + 1] = y1;
  y[3 * (size_t)row + 2] = y2;
}

__global__ void __launch_bounds__(kT) k_spcg_apply(hdk_vtx x, hdk_csr A, int ns, const double* __restrict__ ef,
                                                   const double* __restrict__ p, double* __restrict__ q,
                                                   double* partial, unsigned int* tickets, hdk_pcg* sts) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int smp = blockIdx.y;
  hdk_pcg* st = sts + smp;
  if (st->cond == 0) return;
  const int sub = threadIdx.x & 7, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0_ = smp * ns, r1_ = r0_ + ns;
  double acc[1] = {0.0};
  for (int rb = r0_ + blockIdx.x * (kT / 8) + 4 * warp; rb < r1_; rb += kSRB * (kT / 8)) {
    const int row = rb + (lane >> 3);
    const bool live = row < r1_;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const int e = live ? __ldg(x.pinc_off + row + 1) : 0;
    for (int j = (live ? __ldg(x.pinc_off + row) : 0) + sub; j < e; j += 8) {
      const double* f = ef + 3 * (size_t)j;
      c0 += __ldg(f);
      c1 += __ldg(f + 1);
      c2 += __ldg(f + 2);
    }
    const int ke = live ? __ldg(A.off + row + 1) : 0;
    for (int k = (live ? __ldg(A.off + row) : 0) + sub; k < ke; k += 8) {
      const double w = __ldg(A.val + k);
      const double* v = p + 3 * (size_t)__ldg(A.col + k);
      a0 += w * v[0];
      a1 += w * v[1];
      a2 += w * v[2];
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      c0 += __shfl_xor_sync(0xffffffffu, c0, o);
      c1 += __shfl_xor_sync(0xffffffffu, c1, o);
      c2 += __shfl_xor_sync(0xffffffffu, c2, o);
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (sub == 0 && live) {
      const double q0 = a0 - c0, q1 = a1 - c1, q2 = a2 - c2;
      double* qr = q + 3 * (size_t)row;
      qr[0] = q0;
      qr[1] = q1;
      qr[2] = q2;
      const double* pr = p + 3 * (size_t)row;
      acc[0] += (pr[0] * q0 + pr[1] * q1) + pr[2] * q2;
    }
  }
  double* part = partial + (size_t)smp * HDK_SEG_PSTRIDE;
  block_store_rb<1>(acc, part);
  if (!last_block(tickets + smp)) return;
  if (threadIdx.x >= 32) return;
  const double pq = fold_rb(part, 0);
  if (threadIdx.x != 0) return;
  st->pq = pq;
  if (!(pq > 0.0)) {
    st->err = -1;
    st->cond = 0;
  } else {
    st->alpha = st->rz / pq;
  }
}

__global__ void k_spcg_xr(int n3s, int n3, double* __restrict__ x, double* __restrict__ r,
                          const double* __restrict__ p, const double* __restrict__ q, const hdk_pcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const hdk_pcg& c = st[i / n3s];
  if (c.cond == 0) return;
  const double a = c.alpha;
  x[i] += a * p[i];
  r[i] -= a * q[i];
}

__global__ void __launch_bounds__(kT) k_spcg_rz(int n3s, const double* __restrict__ r, const double* __restrict__ z,
                                                const double* __restrict__ x, double* partial, unsigned int* tickets,
                                                hdk_pcg* sts) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int smp = blockIdx.y;
  hdk_pcg* st = sts + smp;
  if (st->cond == 0) return;
  double acc[3] = {0.0, 0.0, 0.0};
  const int i0 = smp * n3s, i1 = i0 + n3s;
  for (int i = i0 + blockIdx.x * kT + threadIdx.x; i < i1; i += kSRB * kT) {
    const double zi = z[i], t = x[i] + zi;
    acc[0] += r[i] * zi;
    acc[1] += zi * zi;
    acc[2] += t * t;
  }
  double* part = partial + (size_t)smp * HDK_SEG_PSTRIDE;
  block_store_rb<3>(acc, part);
  if (!last_block(tickets + smp)) return;
  if (threadIdx.x >= 32) return;
  const double rz = fold_rb(part, 0), zz = fold_rb(part, 1), tt = fold_rb(part, 2);
  if (threadIdx.x != 0) return;
  const int it = st->iter + 1;
  st->iter = it;
  const bool done = sqrt(zz) <= st->tol * fmax(sqrt(tt), 1e-30);
  st->beta = st->rz > 0.0 && it > 1 ? rz / st->rz : 0.0;
  st->rz = rz;
  st->done = done ? 1 : 0;
  if (!done && it >= st->k_max) st->err = 10;
  if (!isfinite(rz)) st->err = 10;
  st->cond = (!done && st->err == 0) ? 1 : 0;
}

// p = z + beta p per sample; block 0 first publishes the OR of the samples'
// conditions (run flag + WHILE condition).
__global__ void k_spcg_p(int n3s, int n3, const double* __restrict__ z, double* __restrict__ p,
                         double* __restrict__ pv, const int* __restrict__ p2v, const hdk_pcg* st, int count, int* any,
                         cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = i / 3;
  const int vrow = i < n3 ? __ldg(p2v + row) : 0;  // static: before the wait
  hdk::pdl_wait();
  if (blockIdx.x == 0) {
    int on = 0;
    for (int s = threadIdx.x; s < count; s += blockDim.x) on |= (st[s].cond != 0 && st[s].err == 0) ? 1 : 0;
    const int a = __syncthreads_or(on);
    if (threadIdx.x == 0) {
      *any = a;
      if (use_handle) cudaGraphSetConditional(handle, a);
    }
  }
  if (i >= n3) return;
  const hdk_pcg& c = st[i / n3s];
  if (c.cond == 0) return;
  const double v = z[i] + c.beta * p[i];
  p[i] = v;
  pv[3 * (size_t)vrow + (i - 3 * row)] = v;
}

}  // namespace

extern "C" {

HDK_API int hdk_spcg_init(hdk_pcg* st, int count, double tol, int k_max, int* any, void* stream) {
  hdk::launch(k_spcg_init, dim3(1), dim3(256), 0, S(stream), st, count, tol, k_max, any);
  return last();
}
HDK_API int hdk_spcg_spmv(const hdk_csr* a, int ns, const double* p, double* y, const hdk_pcg* st, void* stream) {
  hdk::launch(k_spcg_spmv, dim3(nb(a->rows)), dim3(256), 0, S(stream), *a, ns, p, y, st);
  return last();
}
HDK_API int hdk_spcg_apply(const hdk_vtx* x, const hdk_csr* a, int ns, int count, const double* ef_sorted,
                           const double* p, double* q, double* partial, unsigned int* tickets, hdk_pcg* st,
                           void* stream) {
  if (!x->pinc_off) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_spcg_apply, dim3(kSRB, count), dim3(kT), 0, S(stream), *x, *a, ns, ef_sorted, p, q, partial, tickets,
              st);
  return last();
}
HDK_API int hdk_spcg_xr(int n3s, int n3, double* x, double* r, const double* p, const double* q, const hdk_pcg* st,
                        void* stream) {
  hdk::launch(k_spcg_xr, dim3(nb(n3)), dim3(256), 0, S(stream), n3s, n3, x, r, p, q, st);
  return last();
}
HDK_API int hdk_spcg_rz(int n3s, int count, const double* r, const double* z, const double* x, double* partial,
                        unsigned int* tickets, hdk_pcg* st, void* stream) {
  hdk::launch(k_spcg_rz, dim3(kSRB, count), dim3(kT), 0, S(stream), n3s, r, z, x, partial, tickets, st);
  return last();
}
HDK_API int hdk_spcg_p(int n3s, int n3, const double* z, double* p, double* pv, const int* p2v, const hdk_pcg* st,
                       int count, int* any, unsigned long long cond_handle, void* stream) {
  hdk::launch(k_spcg_p, dim3(nb(n3)), dim3(256), 0, S(stream), n3s, n3, z, p, pv, p2v, st, count, any,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle ? 1 : 0);
  return last();
}

}  // extern "C"

// ---- contact-adjoint columns: one CG per column, all columns per launch -------
// Column c's vectors (elimination order) at base + c n3 (n3 = 3 n); its
// direction by vertex at pv + c n3v; its sorted element forces at
// ef + c ef_stride; z = A^{-1} r is folded per column from the multi-column
// solve's tile partials (part2 + c part2_stride, as the backbone dots fold t).
namespace {

__global__ void k_cpcg_spmv(hdk_csr A, int n3, const double* __restrict__ p, double* __restrict__ y,
                            const hdk_pcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int c = blockIdx.y;
  if (st[c].cond == 0) return;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.rows) return;
  const double* pc = p + (size_t)c * n3;
  double y0 = 0.0, y1 = 0.0, y2 = 0.0;
  for (int k = A.off[row]; k < A.off[row + 1]; ++k) {
    const double w = A.val[k];
    const double* v = pc + 3 * (size_t)A.col[k];
    y0 += w * v[0];
    y1 += w * v[1];
    y2 += w * v[2];
  }
  double* yc = y + (size_t)c * n3 + 3 * (size_t)row;
  yc[0] = y0;
  yc[1] = y1;
  yc[2] = y2;
}

// Column reductions over a grid that covers the rows once (no grid-stride
// loop: at one block per SM-slot the columns' CG stages are latency-bound):
// block b of column c stores quantity q at partial[c pstride + q nb + b];
// the column's last block folds its nb partials in fixed order.
__device__ __forceinline__ double fold_nb(const double* partial, int nb) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += partial[b];
  return warp_sum(s);
}

template <int NQ>
__device__ __forceinline__ void block_store_nb(const double (&v)[NQ], double* partial, int nb) {
  __shared__ double sm[kT / 32][NQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double s = warp_sum(v[q]);
    if (lane == 0) sm[warp][q] = s;
  }
  __syncthreads();
  if (threadIdx.x < NQ) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) s += sm[w][threadIdx.x];
    partial[threadIdx.x * nb + blockIdx.x] = s;
  }
}

// q = A p - gather(B p) per column and p.q; 8 lanes per row, 32 rows per block.
template <bool kReduce>
__global__ void __launch_bounds__(kT) k_cpcg_apply(hdk_vtx x, hdk_csr A, int n3, const double* __restrict__ ef,
                                                   size_t ef_stride, const double* __restrict__ p,
                                                   double* __restrict__ q, double* partial, size_t pstride,
                                                   unsigned int* tickets, hdk_pcg* sts) {
  // the row's static index ranges and its first entry of A before the PDL
  // wait (they do not depend on the previous kernel)
  hdk::pdl_trigger();
  const int c = blockIdx.y;
  const int sub = threadIdx.x & 7;
  const int row = blockIdx.x * (kT / 8) + (threadIdx.x >> 3);
  const bool live = row < x.n;
  const int jb = live ? __ldg(x.pinc_off + row) : 0, e = live ? __ldg(x.pinc_off + row + 1) : 0;
  const int kb = live ? __ldg(A.off + row) : 0, ke = live ? __ldg(A.off + row + 1) : 0;
  const bool has0 = kb + sub < ke;
  const double w0 = has0 ? __ldg(A.val + kb + sub) : 0.0;
  const int col0 = has0 ? __ldg(A.col + kb + sub) : 0;
  hdk::pdl_wait();
  hdk_pcg* st = sts + c;
  if (st->cond == 0) return;
  const double* efc = ef + c * ef_stride;
  const double* pc = p + (size_t)c * n3;
  double* qc = q + (size_t)c * n3;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int j = jb + sub; j < e; j += 8) {
    const double* f = efc + 3 * (size_t)j;
    c0 += __ldg(f);
    c1 += __ldg(f + 1);
    c2 += __ldg(f + 2);
  }
  if (has0) {
    const double* v = pc + 3 * (size_t)col0;
    a0 += w0 * v[0];
    a1 += w0 * v[1];
    a2 += w0 * v[2];
  }
  for (int k = kb + sub + 8; k < ke; k += 8) {
    const double w = __ldg(A.val + k);
    const double* v = pc + 3 * (size_t)__ldg(A.col + k);
    a0 += w * v[0];
    a1 += w * v[1];
    a2 += w * v[2];
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    c0 += __shfl_xor_sync(0xffffffffu, c0, o);
    c1 += __shfl_xor_sync(0xffffffffu, c1, o);
    c2 += __shfl_xor_sync(0xffffffffu, c2, o);
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  double acc[1] = {0.0};
  if (sub == 0 && live) {
    const double q0 = a0 - c0, q1 = a1 - c1, q2 = a2 - c2;
    double* qr = qc + 3 * (size_t)row;
    qr[0] = q0;
    qr[1] = q1;
    qr[2] = q2;
    const double* pr = pc + 3 * (size_t)row;
    acc[0] = (pr[0] * q0 + pr[1] * q1) + pr[2] * q2;
  }
  if (!kReduce) return;
  double* part = partial + (size_t)c * pstride;
  const int nb = gridDim.x;
  block_store_nb<1>(acc, part, nb);
  if (!last_block(tickets + c)) return;
  if (threadIdx.x >= 32) return;
  const double pq = fold_nb(part, nb);
  if (threadIdx.x != 0) return;
  st->pq = pq;
  if (!(pq > 0.0)) {
    st->err = -1;
    st->cond = 0;
  } else {
    st->alpha = st->rz / pq;
  }
}

// Profiling: per-column CG coefficients (alpha_k, beta_k) of the columns' CG
// (the Lanczos matrix of A^{-1}(A - B), HETERODYN_CG_TRACE); null = off.
__device__ double* g_cpcg_trace = nullptr;
constexpr int kCgTraceIters = 512;

// z = A^{-1} r folded per column from the multi-column solve's tile partials
// (the fold of hdk_bb_dots), then r.z, the stopping test and beta.  One
// element per thread.
__global__ void __launch_bounds__(kT) k_cpcg_rz(hdk_factor f, size_t part2_stride, const double* __restrict__ r,
                                                double* __restrict__ z, const double* __restrict__ x, double* partial,
                                                size_t pstride, unsigned int* tickets, hdk_pcg* sts) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int c = blockIdx.y;
  hdk_pcg* st = sts + c;
  if (st->cond == 0) return;
  const size_t n3 = 3 * (size_t)f.n;
  const double* p2 = f.part2 + c * part2_stride;
  double acc[3] = {0.0, 0.0, 0.0};
  const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
  if (i < n3) {
    const double* rc = r + c * n3;
    const double* xc = x + c * n3;
    double* zc = z + c * n3;
    const int col = static_cast<int>(i / 3), a = static_cast<int>(i - 3 * (size_t)col);
    const int tile = col >> 8;
    const int tb0 = __ldg(f.tile_cta2 + 2 * tile), tb1 = __ldg(f.tile_cta2 + 2 * tile + 1);
    const size_t base = (size_t)(tile + tb0) * 256 + (col & 255);
    double zi = 0.0;
    for (int b = 0; b <= tb1 - tb0; ++b) zi += __ldg(p2 + 3 * (base + 256 * (size_t)b) + a);
    zc[i] = zi;
    const double t = xc[i] + zi;
    acc[0] = rc[i] * zi;
    acc[1] = zi * zi;
    acc[2] = t * t;
  }
  double* part = partial + (size_t)c * pstride;
  const int nb = gridDim.x;
  block_store_nb<3>(acc, part, nb);
  if (!last_block(tickets + c)) return;
  if (threadIdx.x >= 32) return;
  const double rz = fold_nb(part, nb), zz = fold_nb(part + nb, nb), tt = fold_nb(part + 2 * nb, nb);
  if (threadIdx.x != 0) return;
  const int it = st->iter + 1;
  st->iter = it;
  const bool done = sqrt(zz) <= st->tol * fmax(sqrt(tt), 1e-30);
  st->beta = st->rz > 0.0 && it > 1 ? rz / st->rz : 0.0;
  if (double* tr = g_cpcg_trace; tr && it > 1 && it - 2 < kCgTraceIters) {
    tr[2 * ((size_t)c * kCgTraceIters + it - 2)] = st->alpha;
    tr[2 * ((size_t)c * kCgTraceIters + it - 2) + 1] = st->beta;
  }
  st->rz = rz;
  st->done = done ? 1 : 0;
  if (!done && it >= st->k_max) st->err = 10;
  if (!isfinite(rz)) st->err = 10;
  st->cond = (!done && st->err == 0) ? 1 : 0;
}

// p = z + beta p per column and by vertex; block (0, 0) publishes the OR of
// the columns' conditions (the multi-column solve's run flag, the WHILE condition).
__global__ void k_cpcg_p(int n, int nv, const double* __restrict__ z, double* __restrict__ p, double* __restrict__ pv,
                         const int* __restrict__ p2v, const hdk_pcg* st, int count, int* any,
                         cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int c = blockIdx.y;
  if (blockIdx.x == 0 && c == 0) {
    int on = 0;
    for (int s = threadIdx.x; s < count; s += blockDim.x) on |= (st[s].cond != 0 && st[s].err == 0) ? 1 : 0;
    const int a = __syncthreads_or(on);
    if (threadIdx.x == 0) {
      *any = a;
      if (use_handle) cudaGraphSetConditional(handle, a);
    }
  }
  if (st[c].cond == 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n3 = 3 * n;
  if (i >= n3) return;
  const double b = st[c].beta;
  const size_t k = (size_t)c * n3 + i;
  const double v = z[k] + b * p[k];
  p[k] = v;
  const int row = i / 3;
  pv[(size_t)c * 3 * nv + 3 * (size_t)__ldg(p2v + row) + (i - 3 * row)] = v;
}

// x_c + z_c by vertex into each column's vertex-order vector (fixed rows untouched).
__global__ void k_cpcg_final(int n, int nv, const double* __restrict__ x, const double* __restrict__ z,
                             double* __restrict__ xv, const int* __restrict__ p2v) {
  const int c = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * n) return;
  const size_t k = (size_t)c * 3 * n + i;
  const int row = i / 3;
  xv[(size_t)c * 3 * nv + 3 * (size_t)__ldg(p2v + row) + (i - 3 * row)] = x[k] + z[k];
}

}  // namespace

extern "C" {

HDK_API int hdk_cpcg_spmv(const hdk_csr* a, int columns, const double* p, double* y, const hdk_pcg* st,
                          void* stream) {
  hdk::launch(k_cpcg_spmv, dim3(nb(a->rows), columns), dim3(256), 0, S(stream), *a, 3 * a->rows, p, y, st);
  return last();
}
HDK_API int hdk_set_cpcg_trace(double* const* trace, void* stream) {  // trace: pinned host cell
  return static_cast<int>(cudaMemcpyToSymbolAsync(g_cpcg_trace, trace, sizeof(double*), 0, cudaMemcpyHostToDevice,
                                                  static_cast<cudaStream_t>(stream)));
}
HDK_API size_t hdk_cpcg_partial_stride(int n) {
  const size_t apply_blocks = (static_cast<size_t>(n) + kT / 8 - 1) / (kT / 8);
  const size_t rz_blocks = (3 * static_cast<size_t>(n) + kT - 1) / kT;
  return 3 * (apply_blocks > rz_blocks ? apply_blocks : rz_blocks);
}
HDK_API int hdk_cpcg_apply(const hdk_vtx* x, const hdk_csr* a, int columns, const double* ef_sorted,
                           size_t ef_stride, const double* p, double* q, double* partial, size_t pstride,
                           unsigned int* tickets, hdk_pcg* st, void* stream) {
  if (!x->pinc_off) return static_cast<int>(cudaErrorInvalidValue);
  const int nbx = (x->n + kT / 8 - 1) / (kT / 8);
  hdk::launch(k_cpcg_apply<true>, dim3(nbx > 0 ? nbx : 1, columns), dim3(kT), 0, S(stream), *x, *a, 3 * x->n,
              ef_sorted, ef_stride, p, q, partial, pstride, tickets, st);
  return last();
}
HDK_API int hdk_cpcg_apply_q(const hdk_vtx* x, const hdk_csr* a, int columns, const double* ef_sorted,
                             size_t ef_stride, const double* p, double* q, hdk_pcg* st, void* stream) {
  if (!x->pinc_off) return static_cast<int>(cudaErrorInvalidValue);
  const int nbx = (x->n + kT / 8 - 1) / (kT / 8);
  hdk::launch(k_cpcg_apply<false>, dim3(nbx > 0 ? nbx : 1, columns), dim3(kT), 0, S(stream), *x, *a, 3 * x->n,
              ef_sorted, ef_stride, p, q, static_cast<double*>(nullptr), size_t{0}, static_cast<unsigned int*>(nullptr),
              st);
  return last();
}
HDK_API int hdk_cpcg_rz(const hdk_factor* f, int columns, const double* r, double* z, const double* x,
                        double* partial, size_t pstride, unsigned int* tickets, hdk_pcg* st, void* stream) {
  if (!f->tile_cta2) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_cpcg_rz, dim3(nb(3LL * f->n), columns), dim3(kT), 0, S(stream), *f, hdk_factor_part2_stride(f), r, z,
              x, partial, pstride, tickets, st);
  return last();
}
HDK_API int hdk_cpcg_p(int n, int nv, int columns, const double* z, double* p, double* pv, const int* p2v,
                       const hdk_pcg* st, int* any, unsigned long long cond_handle, void* stream) {
  hdk::launch(k_cpcg_p, dim3(nb(3LL * n), columns), dim3(256), 0, S(stream), n, nv, z, p, pv, p2v, st, columns, any,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle ? 1 : 0);
  return last();
}
HDK_API int hdk_cpcg_final(int n, int nv, int columns, const double* x, const double* z, double* xv, const int* p2v,
                           void* stream) {
  hdk::launch(k_cpcg_final, dim3(nb(3LL * n), columns), dim3(256), 0, S(stream), n, nv, x, z, xv, p2v);
  return last();
}

}  // extern "C"

// ---- block CG over a batch of contact-adjoint columns -------------------------
// O'Leary's block PCG on (A - B) X = J with the preconditioner A (the
// multi-column solve): the batch's m columns share one block Krylov space,
// so the slow modes of A^{-1}(A - B) that every column meets (the columns'
// Lanczos spectra coincide) are resolved once for the batch.
//   Q = (A - B) P;  alpha = (P^T Q)^{-1} (Z^T R);  X += P alpha;  R -= Q alpha
//   Z = A^{-1} R;   beta = (Z^T R)_old^{-1} (Z^T R);  P = Z + P beta
// The stopping test is the reference's per column (||z_c|| <= tol ||x_c +
// z_c||, backward.cpp:170-204), required of all m columns at the same
// iteration; the columns return x_c + z_c.  The m x m algebra (Cholesky of
// the two Gram matrices) runs in the last block of the reductions; a pivot
// that is not positive ends the block with err = -1.
namespace {

constexpr int kBC = 8;                    // columns per batch (HDK_BB_COLUMNS)
constexpr int kGram = kBC * (kBC + 1) / 2;  // 36: the upper triangle of a symmetric 8 x 8
constexpr int kZq = kGram + 2 * kBC;      // Z^T R triangle + ||z_c||^2 + ||x_c + z_c||^2

__device__ __forceinline__ int tri(int j, int c) { return c * (c + 1) / 2 + j; }  // j <= c

// out = A^{-1} B for m x m symmetric positive definite A, by the whole block
// in shared memory (row r, column c at [r * 8 + c]; entries outside m x m
// ignored): Cholesky column by column (threads over the trailing entries),
// then the m right-hand sides' triangular solves one per thread.  Returns
// false (in every thread) if a pivot is not positive relative to the
// largest diagonal.  A and B are overwritten.
__device__ bool spd_solve8_block(double* a, double* b, int m, double* out) {
  __shared__ int ok;
  __shared__ double dmax;
  const int t = threadIdx.x;
  if (t == 0) {
    double d = 0.0;
    for (int i = 0; i < m; ++i) d = fmax(d, a[i * 8 + i]);
    dmax = d;
    ok = 1;
  }
  __syncthreads();
  for (int k = 0; k < m; ++k) {  // L overwrites the lower triangle of a
    if (t == 0) {
      const double d = a[k * 8 + k];
      if (!(d > 1e-14 * dmax)) ok = 0;
      a[k * 8 + k] = sqrt(fmax(d, 0.0));
    }
    __syncthreads();
    if (!ok) return false;
    const double lkk = a[k * 8 + k];
    if (t > k && t < m) a[t * 8 + k] /= lkk;
    __syncthreads();
    const int i = k + 1 + t / 8, j = k + 1 + t % 8;  // trailing update a[i][j] -= l_ik l_jk, j <= i
    if (t < 64 && i < m && j <= i) a[i * 8 + j] -= a[i * 8 + k] * a[j * 8 + k];
    __syncthreads();
  }
  if (t < m) {  // column t of B: L y = b, L^T x = y
    double y[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r < m) {
        double v = b[r * 8 + t];
        for (int q = 0; q < r; ++q) v -= a[r * 8 + q] * y[q];
        y[r] = v / a[r * 8 + r];
      }
    }
#pragma unroll
    for (int r = 7; r >= 0; --r) {
      if (r < m) {
        double v = y[r];
        for (int q = r + 1; q < m; ++q) v -= a[q * 8 + r] * y[q];
        y[r] = v / a[r * 8 + r];
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) out[r * 8 + t] = r < m ? y[r] : 0.0;
  } else if (t < 8) {
#pragma unroll
    for (int r = 0; r < 8; ++r) out[r * 8 + t] = 0.0;
  }
  __syncthreads();
  return true;
}

template <int NQ>
__device__ __forceinline__ void block_store_many(const double (&v)[NQ], double* partial, int nb) {
  __shared__ double sm[kT / 32][NQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double s = warp_sum(v[q]);
    if (lane == 0) sm[warp][q] = s;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < NQ; q += kT) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) s += sm[w][q];
    partial[(size_t)q * nb + blockIdx.x] = s;
  }
}

// Fixed-order fold of NQ quantities' nb block partials into red[] by the
// whole (last) block: warp w folds quantities w, w + 8, ... with all of its
// loads issued before the shuffle trees (a serial per-quantity fold by one
// warp paid one L2 round trip per quantity: ~50 us for the 52 of k_bcg_zfold).
template <int NQ>
__device__ __forceinline__ void fold_many(const double* partial, int nb, double* red) {
  constexpr int W = kT / 32, PER = (NQ + W - 1) / W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int q = warp + W * k;
    s[k] = 0.0;
    if (q < NQ)
      for (int b = lane; b < nb; b += 32) s[k] += partial[(size_t)q * nb + b];
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const double v = warp_sum(s[k]);
    const int q = warp + W * k;
    if (lane == 0 && q < NQ) red[q] = v;
  }
  __syncthreads();
}

__global__ void k_bcg_init(hdk_bcg* st, const int* m, double tol, int k_max, int* any, hdk_pcg* cst, int cst_count) {
  const int mm = *m;
  if (threadIdx.x == 0) {
    st->m = mm;
    st->tol = tol;
    st->iter = 0;
    st->k_max = k_max;
    st->err = 0;
    st->cond = 1;
    st->done = 0;
    *any = 1;
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) st->rz[i] = st->rz_old[i] = st->g[i] = st->alpha[i] = st->beta[i] = 0.0;
  for (int c = threadIdx.x; c < cst_count; c += blockDim.x) {  // the per-column run flags of B p and q
    cst[c].cond = c < mm ? 1 : 0;
    cst[c].err = 0;
  }
}

// G = P^T Q (upper triangle), then alpha = G^{-1} (Z^T R) in the last block.
__global__ void __launch_bounds__(kT) k_bcg_gram_pq(int n3, const double* __restrict__ p, const double* __restrict__ q,
                                                    double* partial, unsigned int* ticket, hdk_bcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (st->cond == 0) return;
  const int m = st->m;
  const int i = blockIdx.x * kT + threadIdx.x;
  double acc[kGram];
#pragma unroll
  for (int k = 0; k < kGram; ++k) acc[k] = 0.0;
  if (i < n3) {
    double pv[kBC], qv[kBC];
#pragma unroll
    for (int c = 0; c < kBC; ++c) {
      pv[c] = c < m ? p[(size_t)c * n3 + i] : 0.0;
      qv[c] = c < m ? q[(size_t)c * n3 + i] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < kBC; ++c)
#pragma unroll
      for (int j = 0; j <= c; ++j) acc[tri(j, c)] = pv[j] * qv[c];
  }
  const int nb = gridDim.x;
  block_store_many<kGram>(acc, partial, nb);
  if (!last_block(ticket)) return;
  __shared__ double red[kGram];
  fold_many<kGram>(partial, nb, red);
  __shared__ double g[64], rz[64];
  if (threadIdx.x < 64) {
    const int j = threadIdx.x >> 3, c = threadIdx.x & 7;
    const bool in = j < m && c < m;
    g[threadIdx.x] = in ? red[j <= c ? tri(j, c) : tri(c, j)] : 0.0;
    st->g[threadIdx.x] = g[threadIdx.x];
    rz[threadIdx.x] = st->rz[threadIdx.x];
  }
  __syncthreads();
  if (!spd_solve8_block(g, rz, m, st->alpha) && threadIdx.x == 0) {
    st->err = -1;
    st->cond = 0;
  }
}

// X += P alpha, R -= Q alpha (column c: sum over j of column j times alpha[j][c]).
__global__ void k_bcg_xr(int n3, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                         const double* __restrict__ q, const hdk_bcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (st->cond == 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const int m = st->m;
  double pv[kBC], qv[kBC];
#pragma unroll
  for (int j = 0; j < kBC; ++j) {
    pv[j] = j < m ? p[(size_t)j * n3 + i] : 0.0;
    qv[j] = j < m ? q[(size_t)j * n3 + i] : 0.0;
  }
#pragma unroll
  for (int c = 0; c < kBC; ++c) {
    if (c >= m) break;
    double dx = 0.0, dr = 0.0;
#pragma unroll
    for (int j = 0; j < kBC; ++j) {
      const double a = st->alpha[j * 8 + c];
      dx += pv[j] * a;
      dr += qv[j] * a;
    }
    x[(size_t)c * n3 + i] += dx;
    r[(size_t)c * n3 + i] -= dr;
  }
}

// Z = A^{-1} R folded from the multi-column solve's tile partials; Z^T R,
// ||z_c||^2, ||x_c + z_c||^2; in the last block the per-column stopping
// tests and beta = (Z^T R)_old^{-1} (Z^T R).
__global__ void __launch_bounds__(kT) k_bcg_zfold(hdk_factor f, size_t part2_stride, const double* __restrict__ r,
                                                  double* __restrict__ z, const double* __restrict__ x, double* partial,
                                                  unsigned int* ticket, hdk_bcg* st) {
  hdk::pdl_trigger();
  const size_t n3 = 3 * (size_t)f.n;
  const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
  const size_t ii = i < n3 ? i : 0;  // the tile-partial range is static: before the wait
  const int col = static_cast<int>(ii / 3), a = static_cast<int>(ii - 3 * (size_t)col);
  const int tile = col >> 8;
  const int tb0 = __ldg(f.tile_cta2 + 2 * tile), tb1 = __ldg(f.tile_cta2 + 2 * tile + 1);
  hdk::pdl_wait();
  if (st->cond == 0) return;
  const int m = st->m;
  double acc[kZq];
#pragma unroll
  for (int k = 0; k < kZq; ++k) acc[k] = 0.0;
  if (i < n3) {
    const size_t base = (size_t)(tile + tb0) * 256 + (col & 255);
    // every column's loads before any store: the z stores may alias the
    // solve's partials as far as the compiler knows, so a store between
    // two columns' folds serialised eight L2 round trips (51.7 us)
    double zv[kBC], rv[kBC], xv[kBC];
    const int nt = tb1 - tb0;
#pragma unroll
    for (int c = 0; c < kBC; ++c) {
      zv[c] = 0.0;
      rv[c] = 0.0;
      xv[c] = 0.0;
      if (c < m) {
        const double* p2 = f.part2 + c * part2_stride + 3 * base + a;
        double zi = __ldg(p2);
        if (nt >= 1) zi += __ldg(p2 + 3 * 256);
        for (int b = 2; b <= nt; ++b) zi += __ldg(p2 + 3 * 256 * (size_t)b);
        zv[c] = zi;
        rv[c] = r[c * n3 + i];
        xv[c] = x[c * n3 + i];
      }
    }
#pragma unroll
    for (int c = 0; c < kBC; ++c)
      if (c < m) {
        z[c * n3 + i] = zv[c];
        const double t = xv[c] + zv[c];
        acc[kGram + c] = zv[c] * zv[c];
        acc[kGram + kBC + c] = t * t;
      }
#pragma unroll
    for (int c = 0; c < kBC; ++c)
#pragma unroll
      for (int j = 0; j <= c; ++j) acc[tri(j, c)] = zv[j] * rv[c];
  }
  const int nb = gridDim.x;
  block_store_many<kZq>(acc, partial, nb);
  if (!last_block(ticket)) return;
  __shared__ double red[kZq];
  fold_many<kZq>(partial, nb, red);
  const int it = st->iter + 1;
  bool all = true, finite = true;
  for (int c = 0; c < m; ++c) {
    const double zz = red[kGram + c], tt = red[kGram + kBC + c];
    all = all && sqrt(zz) <= st->tol * fmax(sqrt(tt), 1e-30);
    finite = finite && isfinite(zz) && isfinite(tt);
  }
  __shared__ double rz_new[64], a_old[64], rz_rhs[64];
  if (threadIdx.x < 64) {
    const int j = threadIdx.x >> 3, c = threadIdx.x & 7;
    rz_new[threadIdx.x] = (j < m && c < m) ? red[j <= c ? tri(j, c) : tri(c, j)] : 0.0;
    rz_rhs[threadIdx.x] = rz_new[threadIdx.x];
    a_old[threadIdx.x] = st->rz[threadIdx.x];
  }
  __syncthreads();
  bool ok = true;
  if (it > 1 && !all) ok = spd_solve8_block(a_old, rz_rhs, m, st->beta);  // beta = RZ_old^{-1} RZ
  if (threadIdx.x < 64) {
    st->rz_old[threadIdx.x] = st->rz[threadIdx.x];
    st->rz[threadIdx.x] = rz_new[threadIdx.x];
  }
  if (threadIdx.x != 0) return;
  st->iter = it;
  if (!ok) {
    st->err = -1;
    st->cond = 0;
    return;
  }
  st->done = all ? 1 : 0;
  if (!finite || (!all && it >= st->k_max)) st->err = 10;
  st->cond = (!all && st->err == 0) ? 1 : 0;
}

// P = Z + P beta (P = Z after the first solve) and P by vertex; block 0
// publishes the run flag / WHILE condition.
__global__ void k_bcg_p(int n, int nv, const double* __restrict__ z, double* __restrict__ p, double* __restrict__ pv,
                        const int* __restrict__ p2v, const hdk_bcg* st, int* any, const hdk_defl* d,
                        const double* __restrict__ w, cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_trigger();
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int vrow0 = i0 < 3 * n ? __ldg(p2v + i0 / 3) : 0;  // static: before the wait
  hdk::pdl_wait();
  const int on = st->cond != 0 && st->err == 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *any = on;
    if (use_handle) cudaGraphSetConditional(handle, on);
  }
  if (!on) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t n3 = 3 * (size_t)n;
  if (i >= (int)n3) return;
  const int m = st->m;
  const bool first = st->iter == 1;
  double old[kBC];
#pragma unroll
  for (int j = 0; j < kBC; ++j) old[j] = (!first && j < m) ? p[j * n3 + i] : 0.0;
  const int row = i / 3;
  const size_t vtx = 3 * (size_t)vrow0 + (i - 3 * row);
  const bool defl = d && d->cols && d->use && d->active;  // P -= W E^{-1} (AW)^T Z
  const int kd = defl ? d->k : 0;
  double wv[kBC];
#pragma unroll
  for (int q = 0; q < kBC; ++q) wv[q] = q < kd ? w[(size_t)q * n3 + i] : 0.0;
#pragma unroll
  for (int c = 0; c < kBC; ++c) {
    if (c >= m) break;
    double v = z[c * n3 + i];
    if (!first) {
#pragma unroll
      for (int j = 0; j < kBC; ++j) v += old[j] * st->beta[j * 8 + c];
    }
#pragma unroll
    for (int q = 0; q < kBC; ++q)
      if (q < kd) v -= wv[q] * d->cm[q * 8 + c];
    p[c * n3 + i] = v;
    pv[(size_t)c * 3 * nv + vtx] = v;
  }
}

}  // namespace

extern "C" {

HDK_API size_t hdk_bcg_partial_doubles(int n) {
  const size_t nb = (3 * static_cast<size_t>(n) + kT - 1) / kT;
  return static_cast<size_t>(kZq) * nb;
}
HDK_API int hdk_bcg_init(hdk_bcg* st, const int* m, double tol, int k_max, int* any, hdk_pcg* cst, int cst_count,
                         void* stream) {
  hdk::launch(k_bcg_init, dim3(1), dim3(64), 0, S(stream), st, m, tol, k_max, any, cst, cst_count);
  return last();
}
HDK_API int hdk_bcg_gram_pq(int n3, const double* p, const double* q, double* partial, unsigned int* ticket,
                            hdk_bcg* st, void* stream) {
  hdk::launch(k_bcg_gram_pq, dim3(nb(n3)), dim3(kT), 0, S(stream), n3, p, q, partial, ticket, st);
  return last();
}
HDK_API int hdk_bcg_xr(int n3, double* x, double* r, const double* p, const double* q, const hdk_bcg* st,
                       void* stream) {
  hdk::launch(k_bcg_xr, dim3(nb(n3)), dim3(256), 0, S(stream), n3, x, r, p, q, st);
  return last();
}
HDK_API int hdk_bcg_zfold(const hdk_factor* f, const double* r, double* z, const double* x, double* partial,
                          unsigned int* ticket, hdk_bcg* st, void* stream) {
  if (!f->tile_cta2) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_bcg_zfold, dim3(nb(3LL * f->n)), dim3(kT), 0, S(stream), *f, hdk_factor_part2_stride(f), r, z, x,
              partial, ticket, st);
  return last();
}
HDK_API int hdk_bcg_p(int n, int nv, const double* z, double* p, double* pv, const int* p2v, hdk_bcg* st, int* any,
                      const hdk_defl* d, const double* w, unsigned long long cond_handle, void* stream) {
  hdk::launch(k_bcg_p, dim3(nb(3LL * n)), dim3(256), 0, S(stream), n, nv, z, p, pv, p2v,
              static_cast<const hdk_bcg*>(st), any, d, w,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle ? 1 : 0);
  return last();
}

}  // extern "C"

// ---- deflated CG for the single backbone ---------------------------------------
// (hdk.h hdk_defl).  Per iteration the r.z kernel also forms d = (AW)^T z
// and mu = E^{-1} d (E = W^T A' W, A' = A - B, Cholesky factor precomputed),
// and the p kernel subtracts W mu: p = z + beta p - W mu.  A recording solve
// (no deflation) keeps its z's and (alpha, beta, r.z) for the host's Ritz
// extraction.  Up to kDK = HDK_DEFL_MAX vectors.
namespace {

constexpr int kDK = HDK_DEFL_MAX;
constexpr int kDq = 3 + kDK;  // r.z, |z|^2, |x + z|^2, (AW_k)^T z

__device__ void chol_solve_l(const double* l, int k, const double* b, double* x) {  // L L^T x = b
  double y[kDK];
  for (int i = 0; i < k; ++i) {
    double v = b[i];
    for (int t = 0; t < i; ++t) v -= l[i * kDK + t] * y[t];
    y[i] = v / l[i * kDK + i];
  }
  for (int i = k - 1; i >= 0; --i) {
    double v = y[i];
    for (int t = i + 1; t < k; ++t) v -= l[t * kDK + i] * y[t];
    y[i] = v / l[i * kDK + i];
  }
  for (int i = 0; i < k; ++i) x[i] = y[i];
}

// E[j][c] = (w_j . aw_c + w_c . aw_j) / 2: kGramSlices blocks per (j <= c)
// pair, the slices folded in fixed order by k_defl_chol.
constexpr int kGramSlices = 16;
__global__ void __launch_bounds__(kT) k_defl_gram(int n3, const double* __restrict__ w, const double* __restrict__ aw,
                                                  double* e, const hdk_defl* d) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (!d->use) return;
  const int k = d->k;
  int j = 0, idx = blockIdx.x;  // pair index -> (j, c), j <= c: ordered by j, then c = j .. kDK - 1
  while (idx >= kDK - j) {
    idx -= kDK - j;
    ++j;
  }
  const int c = j + idx;
  if (j >= k || c >= k) return;
  double acc[1] = {0.0};  // slice blockIdx.y of the pair's dot product
  for (int i = blockIdx.y * kT + threadIdx.x; i < n3; i += kGramSlices * kT)
    acc[0] += 0.5 * (w[(size_t)j * n3 + i] * aw[(size_t)c * n3 + i] + w[(size_t)c * n3 + i] * aw[(size_t)j * n3 + i]);
  __shared__ double sm[kT / 32];
  const double v = warp_sum(acc[0]);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kT / 32; ++q) t += sm[q];
    e[kDK * kDK + (size_t)blockIdx.x * kGramSlices + blockIdx.y] = t;  // slice partials after the matrix
  }
}

// Cholesky of E once per step; active = factor ok.  One warp: lanes fold the
// pairs' slice partials, lane 0 factors in shared memory, lanes 0..k-1 form
// E^{-1} column by column (the per-iteration mu = E^{-1} d becomes a
// mat-vec).  The factor used to live in global memory with one thread
// (52 us a step: every access a dependent global round trip).
__global__ void k_defl_chol(const double* __restrict__ e, hdk_defl* d) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (!d->use) return;
  const int k = d->k, lane = threadIdx.x;
  __shared__ double l[kDK * kDK];
  __shared__ int ok_s;
  for (int q = lane; q < kDK * kDK; q += 32) l[q] = 0.0;
  __syncwarp();
  constexpr int kPairs = kDK * (kDK + 1) / 2;
  for (int pair = lane; pair < kPairs; pair += 32) {
    int pj = 0, idx = pair;  // pair -> (pj, pc), pj <= pc, ordered by pj then pc
    while (idx >= kDK - pj) {
      idx -= kDK - pj;
      ++pj;
    }
    const int pc = pj + idx;
    if (pj >= k || pc >= k) continue;
    double t = 0.0;
    for (int q = 0; q < kGramSlices; ++q) t += e[kDK * kDK + (size_t)pair * kGramSlices + q];
    l[pc * kDK + pj] = t;  // lower triangle (row pc >= column pj)
  }
  __syncwarp();
  if (lane == 0) {
    double dmax = 0.0;
    for (int r = 0; r < k; ++r) dmax = fmax(dmax, l[r * kDK + r]);
    bool ok = k > 0;
    for (int j = 0; j < k && ok; ++j) {
      double dj = l[j * kDK + j];
      for (int t = 0; t < j; ++t) dj -= l[j * kDK + t] * l[j * kDK + t];
      if (!(dj > 1e-12 * dmax)) {
        ok = false;
        break;
      }
      dj = sqrt(dj);
      l[j * kDK + j] = dj;
      for (int r = j + 1; r < k; ++r) {
        double v = l[r * kDK + j];
        for (int t = 0; t < j; ++t) v -= l[r * kDK + t] * l[j * kDK + t];
        l[r * kDK + j] = v / dj;
      }
    }
    ok_s = ok ? 1 : 0;
  }
  __syncwarp();
  const bool ok = ok_s != 0;
  for (int q = lane; q < kDK * kDK; q += 32) d->l[q] = l[q];
  if (ok && lane < kDK) {  // column lane of E^{-1}
    double col[kDK];
#pragma unroll
    for (int r = 0; r < kDK; ++r) col[r] = (r == lane) ? 1.0 : 0.0;
    if (lane < k) chol_solve_l(l, k, col, col);
#pragma unroll
    for (int r = 0; r < kDK; ++r) d->einv[r * kDK + lane] = (r < k && lane < k) ? col[r] : 0.0;
  }
  if (lane == 0) d->active = ok ? 1 : 0;
}

// First iterate: c = E^{-1} W^T r (last block), then (k_defl_correct) x += W c, r -= AW c.
__global__ void __launch_bounds__(kT) k_defl_dots(int n3, const double* __restrict__ r, const double* __restrict__ w,
                                                  double* partial, unsigned int* ticket, hdk_defl* d) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (!d->use || !d->active) return;
  const int k = d->k;
  const int i = blockIdx.x * kT + threadIdx.x;
  double acc[kDK];
#pragma unroll
  for (int c = 0; c < kDK; ++c) acc[c] = (i < n3 && c < k) ? w[(size_t)c * n3 + i] * r[i] : 0.0;
  const int nb = gridDim.x;
  block_store_many<kDK>(acc, partial, nb);
  if (!last_block(ticket)) return;
  __shared__ double red[kDK];
  fold_many<kDK>(partial, nb, red);
  if (threadIdx.x != 0) return;
  double cc[kDK];
  chol_solve_l(d->l, k, red, cc);
  for (int c = 0; c < kDK; ++c) d->c[c] = c < k ? cc[c] : 0.0;
}

__global__ void k_defl_correct(int n3, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ w,
                               const double* __restrict__ aw, const hdk_defl* d) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (!d->use || !d->active) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const int k = d->k;
  double dx = 0.0, dr = 0.0;
#pragma unroll
  for (int c = 0; c < kDK; ++c)
    if (c < k) {
      dx += w[(size_t)c * n3 + i] * d->c[c];
      dr += aw[(size_t)c * n3 + i] * d->c[c];
    }
  x[i] += dx;
  r[i] -= dr;
}

// z from the solve's tile partials, r.z / |z|^2 / |x + z|^2, d = (AW)^T z;
// last block: stopping test, beta, mu = E^{-1} d; recording: z and the
// coefficients into the history.
__global__ void __launch_bounds__(kT) k_dpcg_rz(hdk_factor f, const double* __restrict__ r, double* __restrict__ z,
                                                const double* __restrict__ x, const double* __restrict__ aw,
                                                double* partial, unsigned int* ticket, hdk_pcg* st, hdk_defl* d,
                                                double* __restrict__ zhist, double* hist) {
  // the element's tile-partial range is static: read before the wait
  hdk::pdl_trigger();
  const size_t n3 = 3 * (size_t)f.n;
  const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
  const size_t ii = i < n3 ? i : 0;
  const int col = static_cast<int>(ii / 3), a = static_cast<int>(ii - 3 * (size_t)col);
  const int tile = col >> 8;
  const int tb0 = __ldg(f.tile_cta2 + 2 * tile), tb1 = __ldg(f.tile_cta2 + 2 * tile + 1);
  hdk::pdl_wait();
  if (st->cond == 0) return;
  const bool defl = d->use && d->active;
  const int k = defl ? d->k : 0;
  const int it = st->iter + 1;
  const bool rec = d->rec && it <= d->hcap;
  double acc[kDq];
#pragma unroll
  for (int q = 0; q < kDq; ++q) acc[q] = 0.0;
  if (i < n3) {
    // the loads that do not depend on the fold first, all before the stores
    const double ri = r[i], xi = x[i];
    double awi[kDK];
#pragma unroll
    for (int c = 0; c < kDK; ++c) awi[c] = c < k ? aw[(size_t)c * n3 + i] : 0.0;
    const size_t base = (size_t)(tile + tb0) * 256 + (col & 255);
    double zi = 0.0;
    for (int b = 0; b <= tb1 - tb0; ++b) zi += __ldg(f.part2 + 3 * (base + 256 * (size_t)b) + a);
    z[i] = zi;
    if (rec) zhist[(size_t)(it - 1) * n3 + i] = zi;
    const double t = xi + zi;
    acc[0] = ri * zi;
    acc[1] = zi * zi;
    acc[2] = t * t;
#pragma unroll
    for (int c = 0; c < kDK; ++c) acc[3 + c] = awi[c] * zi;
  }
  const int nb = gridDim.x;
  block_store_many<kDq>(acc, partial, nb);
  if (!last_block(ticket)) return;
  __shared__ double red[kDq];
  fold_many<kDq>(partial, nb, red);
  if (defl && threadIdx.x < kDK) {  // mu = E^{-1} d, one row per thread
    double m = 0.0;
#pragma unroll
    for (int j = 0; j < kDK; ++j) m += d->einv[threadIdx.x * kDK + j] * red[3 + j];
    d->mu[threadIdx.x] = threadIdx.x < k ? m : 0.0;
  }
  if (threadIdx.x != 0) return;
  const double rz = red[0], zz = red[1], tt = red[2];
  st->iter = it;
  const bool done = sqrt(zz) <= st->tol * fmax(sqrt(tt), 1e-30);
  st->beta = st->rz > 0.0 && it > 1 ? rz / st->rz : 0.0;
  if (rec) {
    hist[3 * (it - 1)] = it > 1 ? st->alpha : 0.0;
    hist[3 * (it - 1) + 1] = st->beta;
    hist[3 * (it - 1) + 2] = rz;
  }
  st->rz = rz;
  st->done = done ? 1 : 0;
  if (!done && it >= st->k_max) st->err = 10;
  if (!isfinite(rz)) st->err = 10;
  st->cond = (!done && st->err == 0) ? 1 : 0;
}

// p = z + beta p - W mu, and p by vertex; the WHILE condition.
__global__ void k_dpcg_p(int n, const double* __restrict__ z, double* __restrict__ p, double* __restrict__ pv,
                         const int* __restrict__ p2v, const hdk_pcg* st, const hdk_defl* d,
                         const double* __restrict__ w, cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t n3 = 3 * (size_t)n;
  const int row = i / 3;
  const int vrow = i < (int)n3 ? __ldg(p2v + row) : 0;  // static: before the wait
  hdk::pdl_wait();
  if (use_handle && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(handle, st->cond);
  if (st->cond == 0) return;
  if (i >= (int)n3) return;
  double v = z[i] + st->beta * p[i];
  if (d->use && d->active) {
    const int k = d->k;
#pragma unroll
    for (int c = 0; c < kDK; ++c)
      if (c < k) v -= w[(size_t)c * n3 + i] * d->mu[c];
  }
  p[i] = v;
  pv[3 * (size_t)vrow + (i - 3 * row)] = v;
}

// w_c = sum_j coef[c J + j] zhist_j (the Ritz vectors of a recorded solve).
__global__ void k_ritz_combine(int n3, const double* __restrict__ zhist, const double* __restrict__ coef, int nj,
                               int k, double* __restrict__ w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  double acc[kDK];
#pragma unroll
  for (int c = 0; c < kDK; ++c) acc[c] = 0.0;
  for (int j = 0; j < nj; ++j) {
    const double zj = zhist[(size_t)j * n3 + i];
#pragma unroll
    for (int c = 0; c < kDK; ++c)
      if (c < k) acc[c] += __ldg(coef + c * nj + j) * zj;
  }
#pragma unroll
  for (int c = 0; c < kDK; ++c)
    if (c < k) w[(size_t)c * n3 + i] = acc[c];
}

// Block CG columns: cm[:, c] = E^{-1} Wsrc^T v_c for the batch's columns
// (blockIdx.y = column, its own partials and ticket).
__global__ void __launch_bounds__(kT) k_bdefl_dots(int n3, const double* __restrict__ v,
                                                   const double* __restrict__ wsrc, hdk_defl* d, const hdk_bcg* st,
                                                   double* partial, unsigned int* tickets) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int c = blockIdx.y;
  if (!d->cols || !d->use || !d->active || c >= st->m || st->cond == 0) return;
  const int k = d->k;
  const int i = blockIdx.x * kT + threadIdx.x;
  double acc[kDK];
  const double vi = i < n3 ? v[(size_t)c * n3 + i] : 0.0;
#pragma unroll
  for (int q = 0; q < kDK; ++q) acc[q] = (i < n3 && q < k) ? wsrc[(size_t)q * n3 + i] * vi : 0.0;
  const int nb = gridDim.x;
  double* part = partial + (size_t)c * kDK * nb;
  block_store_many<kDK>(acc, part, nb);
  if (!last_block(tickets + c)) return;
  __shared__ double red[kDK];
  fold_many<kDK>(part, nb, red);
  if (threadIdx.x != 0) return;
  double out[kDK];
  chol_solve_l(d->l, k, red, out);
  for (int q = 0; q < kDK; ++q) d->cm[q * 8 + c] = q < k ? out[q] : 0.0;
}

// X_c += W cm[:, c], R_c -= AW cm[:, c].
__global__ void k_bdefl_correct(int n3, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ w,
                                const double* __restrict__ aw, const hdk_defl* d, const hdk_bcg* st) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (!d->cols || !d->use || !d->active || st->cond == 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const int k = d->k, m = st->m;
  double wv[kDK], av[kDK];
#pragma unroll
  for (int q = 0; q < kDK; ++q) {
    wv[q] = q < k ? w[(size_t)q * n3 + i] : 0.0;
    av[q] = q < k ? aw[(size_t)q * n3 + i] : 0.0;
  }
  for (int c = 0; c < m; ++c) {
    double dx = 0.0, dr = 0.0;
#pragma unroll
    for (int q = 0; q < kDK; ++q) {
      const double cq = d->cm[q * 8 + c];
      dx += wv[q] * cq;
      dr += av[q] * cq;
    }
    x[(size_t)c * n3 + i] += dx;
    r[(size_t)c * n3 + i] -= dr;
  }
}

// W by vertex (the B apply's layout; fixed vertices stay 0).
__global__ void k_scatter_cols(int n, int nv, int kmax, const double* __restrict__ w, double* __restrict__ wv,
                               const int* __restrict__ p2v, const hdk_defl* d) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (!d->use) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t n3 = 3 * (size_t)n;
  if (i >= (int)n3) return;
  const int row = i / 3;
  const size_t vtx = 3 * (size_t)__ldg(p2v + row) + (i - 3 * row);
  for (int c = 0; c < kmax; ++c) wv[(size_t)c * 3 * nv + vtx] = c < d->k ? w[(size_t)c * n3 + i] : 0.0;
}

}  // namespace

extern "C" {

HDK_API size_t hdk_defl_partial_doubles(int n) {
  const size_t nb = (3 * static_cast<size_t>(n) + kT - 1) / kT;
  return std::max(static_cast<size_t>(kDq) * nb, static_cast<size_t>(kDK) * kDK + kDK * (kDK + 1) / 2 * kGramSlices);
}
HDK_API int hdk_defl_gram(int n3, const double* w, const double* aw, double* partial, unsigned int* ticket,
                          hdk_defl* d, void* stream) {
  (void)ticket;
  double* e = partial;  // kDK x kDK
  hdk::launch(k_defl_gram, dim3(kDK * (kDK + 1) / 2, kGramSlices), dim3(kT), 0, S(stream), n3, w, aw, e,
              static_cast<const hdk_defl*>(d));
  hdk::launch(k_defl_chol, dim3(1), dim3(32), 0, S(stream), static_cast<const double*>(e), d);
  return last();
}
HDK_API int hdk_defl_galerkin(int n3, double* x, double* r, const double* w, const double* aw, double* partial,
                              unsigned int* ticket, hdk_defl* d, void* stream) {
  hdk::launch(k_defl_dots, dim3(nb(n3)), dim3(kT), 0, S(stream), n3, static_cast<const double*>(r), w, partial, ticket,
              d);
  hdk::launch(k_defl_correct, dim3(nb(n3)), dim3(256), 0, S(stream), n3, x, r, w, aw, static_cast<const hdk_defl*>(d));
  return last();
}
HDK_API int hdk_dpcg_rz(const hdk_factor* f, const double* r, double* z, const double* x, const double* aw,
                        double* partial, unsigned int* ticket, hdk_pcg* st, hdk_defl* d, double* zhist,
                        double* hist, void* stream) {
  if (!f->tile_cta2) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_dpcg_rz, dim3(nb(3LL * f->n)), dim3(kT), 0, S(stream), *f, r, z, x, aw, partial, ticket, st, d, zhist,
              hist);
  return last();
}
HDK_API int hdk_dpcg_p(int n, const double* z, double* p, double* pv, const int* p2v, const hdk_pcg* st,
                       const hdk_defl* d, const double* w, unsigned long long cond_handle, void* stream) {
  hdk::launch(k_dpcg_p, dim3(nb(3LL * n)), dim3(256), 0, S(stream), n, z, p, pv, p2v, st, d, w,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle ? 1 : 0);
  return last();
}
HDK_API size_t hdk_bdefl_partial_doubles(int n) {
  const size_t nb = (3 * static_cast<size_t>(n) + kT - 1) / kT;
  return static_cast<size_t>(8) * kDK * nb;
}
HDK_API int hdk_bdefl_dots(int n3, const double* v, const double* wsrc, hdk_defl* d, const hdk_bcg* st,
                           double* partial, unsigned int* tickets, void* stream) {
  hdk::launch(k_bdefl_dots, dim3(nb(n3), 8), dim3(kT), 0, S(stream), n3, v, wsrc, d, st, partial, tickets);
  return last();
}
HDK_API int hdk_bdefl_correct(int n3, double* x, double* r, const double* w, const double* aw, const hdk_defl* d,
                              const hdk_bcg* st, void* stream) {
  hdk::launch(k_bdefl_correct, dim3(nb(n3)), dim3(256), 0, S(stream), n3, x, r, w, aw, d, st);
  return last();
}
HDK_API int hdk_ritz_combine(int n3, const double* zhist, const double* coef, int j, int k, double* w, void* stream) {
  k_ritz_combine<<<nb(n3), 256, 0, S(stream)>>>(n3, zhist, coef, j, k, w);
  return last();
}
HDK_API int hdk_scatter_cols(int n, int nv, int k, const double* w, double* wv, const int* p2v, const hdk_defl* d,
                             void* stream) {
  hdk::launch(k_scatter_cols, dim3(nb(3LL * n)), dim3(256), 0, S(stream), n, nv, k, w, wv, p2v, d);
  return last();
}

}  // extern "C"

// ---- deflated CG for the lockstep batch (per sample) ----------------------------
namespace {

constexpr int kSDq = 3 + HDK_DEFL_MAX;

__device__ void chol_solve_s(const double* l, int k, const double* b, double* x) {  // L L^T x = b
  constexpr int K = HDK_DEFL_MAX;
  double y[K];
  for (int i = 0; i < k; ++i) {
    double v = b[i];
    for (int t = 0; t < i; ++t) v -= l[i * K + t] * y[t];
    y[i] = v / l[i * K + i];
  }
  for (int i = k - 1; i >= 0; --i) {
    double v = y[i];
    for (int t = i + 1; t < k; ++t) v -= l[t * K + i] * y[t];
    y[i] = v / l[i * K + i];
  }
  for (int i = 0; i < k; ++i) x[i] = y[i];
}

// E_s[j][c] for every sample: block (pair, sample), fixed-order sums over the sample's range.
__global__ void __launch_bounds__(kT) k_sdefl_gram(int n3s, const double* __restrict__ w, const double* __restrict__ aw,
                                                   const hdk_defl* d, double* e) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  constexpr int K = HDK_DEFL_MAX;
  if (!d->use) return;
  const int k = d->k, smp = blockIdx.y;
  int j = 0, idx = blockIdx.x;
  while (idx >= K - j) {
    idx -= K - j;
    ++j;
  }
  const int c = j + idx;
  if (j >= k || c >= k) return;
  const size_t n3 = (size_t)n3s * gridDim.y, i0 = (size_t)smp * n3s;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n3s; i += kT) {
    const size_t g = i0 + i;
    acc += 0.5 * (w[j * n3 + g] * aw[c * n3 + g] + w[c * n3 + g] * aw[j * n3 + g]);
  }
  __shared__ double sm[kT / 32];
  const double v = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kT / 32; ++q) t += sm[q];
    e[(size_t)smp * K * K + j * K + c] = t;
    e[(size_t)smp * K * K + c * K + j] = t;
  }
}

// One thread per sample: Cholesky of E_s, active_s.
__global__ void k_sdefl_chol(int count, const double* __restrict__ e, const hdk_defl* d, hdk_sdefl* ds) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  constexpr int K = HDK_DEFL_MAX;
  const int smp = blockIdx.x * blockDim.x + threadIdx.x;
  if (smp >= count) return;
  hdk_sdefl* o = ds + smp;
  if (!d->use) {
    o->active = 0;
    return;
  }
  const int k = d->k;
  double* l = o->l;
  const double* es = e + (size_t)smp * K * K;
  for (int q = 0; q < K * K; ++q) l[q] = 0.0;
  for (int r = 0; r < k; ++r)
    for (int c = 0; c <= r; ++c) l[r * K + c] = es[r * K + c];
  double dmax = 0.0;
  for (int r = 0; r < k; ++r) dmax = fmax(dmax, l[r * K + r]);
  bool ok = k > 0;
  for (int j = 0; j < k && ok; ++j) {
    double dj = l[j * K + j];
    for (int t = 0; t < j; ++t) dj -= l[j * K + t] * l[j * K + t];
    if (!(dj > 1e-12 * dmax)) {
      ok = false;
      break;
    }
    dj = sqrt(dj);
    l[j * K + j] = dj;
    for (int r = j + 1; r < k; ++r) {
      double v = l[r * K + j];
      for (int t = 0; t < j; ++t) v -= l[r * K + t] * l[j * K + t];
      l[r * K + j] = v / dj;
    }
  }
  o->active = ok ? 1 : 0;
}

// Galerkin first iterate per sample: c_s = E_s^{-1} W_s^T r_s (grid (kSRB, S)).
__global__ void __launch_bounds__(kT) k_sdefl_dots(int n3s, const double* __restrict__ r, const double* __restrict__ w,
                                                   const hdk_defl* d, hdk_sdefl* ds, double* partial,
                                                   unsigned int* tickets) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  constexpr int K = HDK_DEFL_MAX;
  const int smp = blockIdx.y;
  if (!d->use || !ds[smp].active) return;
  const int k = d->k;
  const size_t n3 = (size_t)n3s * gridDim.y;
  double acc[K];
#pragma unroll
  for (int q = 0; q < K; ++q) acc[q] = 0.0;
  const size_t i0 = (size_t)smp * n3s, i1 = i0 + n3s;
  for (size_t i = i0 + blockIdx.x * kT + threadIdx.x; i < i1; i += (size_t)kSRB * kT) {
    const double ri = r[i];
#pragma unroll
    for (int q = 0; q < K; ++q)
      if (q < k) acc[q] += w[q * n3 + i] * ri;
  }
  double* part = partial + (size_t)smp * HDK_SEG_PSTRIDE;
  block_store_rb<K>(acc, part);
  if (!last_block(tickets + smp)) return;
  if (threadIdx.x >= 32) return;
  double red[K];
#pragma unroll
  for (int q = 0; q < K; ++q) red[q] = fold_rb(part, q);
  if (threadIdx.x != 0) return;
  double cc[K];
  chol_solve_s(ds[smp].l, k, red, cc);
  for (int q = 0; q < K; ++q) ds[smp].c[q] = q < k ? cc[q] : 0.0;
}

__global__ void k_sdefl_correct(int n3s, int n3, double* __restrict__ x, double* __restrict__ r,
                                const double* __restrict__ w, const double* __restrict__ aw, const hdk_defl* d,
                                const hdk_sdefl* ds) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  constexpr int K = HDK_DEFL_MAX;
  if (!d->use) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const hdk_sdefl& o = ds[i / n3s];
  if (!o.active) return;
  const int k = d->k;
  double dx = 0.0, dr = 0.0;
#pragma unroll
  for (int q = 0; q < K; ++q)
    if (q < k) {
      dx += w[(size_t)q * n3 + i] * o.c[q];
      dr += aw[(size_t)q * n3 + i] * o.c[q];
    }
  x[i] += dx;
  r[i] -= dr;
}

// k_spcg_rz plus d_s = (AW_s)^T z_s, mu_s = E_s^{-1} d_s, and the recording.
__global__ void __launch_bounds__(kT) k_sdpcg_rz(int n3s, const double* __restrict__ r, const double* __restrict__ z,
                                                 const double* __restrict__ x, const double* __restrict__ aw,
                                                 double* partial, unsigned int* tickets, hdk_pcg* sts,
                                                 const hdk_defl* d, hdk_sdefl* ds, double* __restrict__ zhist,
                                                 double* hist) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  constexpr int K = HDK_DEFL_MAX;
  const int smp = blockIdx.y;
  hdk_pcg* st = sts + smp;
  if (st->cond == 0) return;
  const bool defl = d->use && ds[smp].active;
  const int k = defl ? d->k : 0;
  const int it = st->iter + 1;
  const bool rec = d->rec && it <= d->hcap;
  const size_t n3 = (size_t)n3s * gridDim.y;
  double acc[kSDq];
#pragma unroll
  for (int q = 0; q < kSDq; ++q) acc[q] = 0.0;
  const size_t i0 = (size_t)smp * n3s, i1 = i0 + n3s;
  for (size_t i = i0 + blockIdx.x * kT + threadIdx.x; i < i1; i += (size_t)kSRB * kT) {
    const double zi = z[i], t = x[i] + zi;
    if (rec) zhist[(size_t)(it - 1) * n3 + i] = zi;
    acc[0] += r[i] * zi;
    acc[1] += zi * zi;
    acc[2] += t * t;
#pragma unroll
    for (int q = 0; q < K; ++q)
      if (q < k) acc[3 + q] += aw[q * n3 + i] * zi;
  }
  double* part = partial + (size_t)smp * HDK_SEG_PSTRIDE;
  block_store_rb<kSDq>(acc, part);
  if (!last_block(tickets + smp)) return;
  if (threadIdx.x >= 32) return;
  double red[kSDq];
#pragma unroll
  for (int q = 0; q < kSDq; ++q) red[q] = fold_rb(part, q);
  if (threadIdx.x != 0) return;
  const double rz = red[0], zz = red[1], tt = red[2];
  st->iter = it;
  const bool done = sqrt(zz) <= st->tol * fmax(sqrt(tt), 1e-30);
  st->beta = st->rz > 0.0 && it > 1 ? rz / st->rz : 0.0;
  if (rec) {
    double* h = hist + (size_t)smp * 3 * d->hcap;
    h[3 * (it - 1)] = it > 1 ? st->alpha : 0.0;
    h[3 * (it - 1) + 1] = st->beta;
    h[3 * (it - 1) + 2] = rz;
  }
  st->rz = rz;
  st->done = done ? 1 : 0;
  if (!done && it >= st->k_max) st->err = 10;
  if (!isfinite(rz)) st->err = 10;
  st->cond = (!done && st->err == 0) ? 1 : 0;
  if (defl) {
    double mu[K];
    chol_solve_s(ds[smp].l, k, red + 3, mu);
    for (int q = 0; q < K; ++q) ds[smp].mu[q] = q < k ? mu[q] : 0.0;
  }
}

// k_spcg_p minus W_s mu_s.
__global__ void k_sdpcg_p(int n3s, int n3, const double* __restrict__ z, double* __restrict__ p,
                          double* __restrict__ pv, const int* __restrict__ p2v, const hdk_pcg* st, int count, int* any,
                          const hdk_defl* d, const hdk_sdefl* ds, const double* __restrict__ w,
                          cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  constexpr int K = HDK_DEFL_MAX;
  if (blockIdx.x == 0) {
    int on = 0;
    for (int s = threadIdx.x; s < count; s += blockDim.x) on |= (st[s].cond != 0 && st[s].err == 0) ? 1 : 0;
    const int a = __syncthreads_or(on);
    if (threadIdx.x == 0) {
      *any = a;
      if (use_handle) cudaGraphSetConditional(handle, a);
    }
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const int smp = i / n3s;
  const hdk_pcg& c = st[smp];
  if (c.cond == 0) return;
  double v = z[i] + c.beta * p[i];
  if (d->use && ds[smp].active) {
    const int k = d->k;
#pragma unroll
    for (int q = 0; q < K; ++q)
      if (q < k) v -= w[(size_t)q * n3 + i] * ds[smp].mu[q];
  }
  p[i] = v;
  const int row = i / 3;
  pv[3 * (size_t)__ldg(p2v + row) + (i - 3 * row)] = v;
}

// w_c[i] = sum_j coef[s][c][j] zhist_j[i], s = sample of i (coefficients zero past a sample's own count).
__global__ void k_sritz_combine(int n3s, int n3, const double* __restrict__ zhist, const double* __restrict__ coef,
                                int jmax, int k, double* __restrict__ w) {
  constexpr int K = HDK_DEFL_MAX;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const double* cs = coef + (size_t)(i / n3s) * K * jmax;
  double acc[K];
#pragma unroll
  for (int q = 0; q < K; ++q) acc[q] = 0.0;
  for (int j = 0; j < jmax; ++j) {
    const double zj = zhist[(size_t)j * n3 + i];
#pragma unroll
    for (int q = 0; q < K; ++q)
      if (q < k) acc[q] += __ldg(cs + q * jmax + j) * zj;
  }
#pragma unroll
  for (int q = 0; q < K; ++q)
    if (q < k) w[(size_t)q * n3 + i] = acc[q];
}

}  // namespace

extern "C" {

HDK_API int hdk_sdefl_gram(int n3s, int count, const double* w, const double* aw, const hdk_defl* d, hdk_sdefl* ds,
                           double* e, void* stream) {
  constexpr int K = HDK_DEFL_MAX;
  hdk::launch(k_sdefl_gram, dim3(K * (K + 1) / 2, count), dim3(kT), 0, S(stream), n3s, w, aw, d, e);
  hdk::launch(k_sdefl_chol, dim3((count + 63) / 64), dim3(64), 0, S(stream), count, static_cast<const double*>(e), d,
              ds);
  return last();
}
HDK_API int hdk_sdefl_galerkin(int n3s, int count, double* x, double* r, const double* w, const double* aw,
                               const hdk_defl* d, hdk_sdefl* ds, double* partial, unsigned int* tickets, void* stream) {
  hdk::launch(k_sdefl_dots, dim3(kSRB, count), dim3(kT), 0, S(stream), n3s, static_cast<const double*>(r), w, d, ds,
              partial, tickets);
  hdk::launch(k_sdefl_correct, dim3(nb(static_cast<long long>(n3s) * count)), dim3(256), 0, S(stream), n3s,
              n3s * count, x, r, w, aw, d, static_cast<const hdk_sdefl*>(ds));
  return last();
}
HDK_API int hdk_sdpcg_rz(int n3s, int count, const double* r, const double* z, const double* x, const double* aw,
                         double* partial, unsigned int* tickets, hdk_pcg* st, const hdk_defl* d, hdk_sdefl* ds,
                         double* zhist, double* hist, void* stream) {
  hdk::launch(k_sdpcg_rz, dim3(kSRB, count), dim3(kT), 0, S(stream), n3s, r, z, x, aw, partial, tickets, st, d, ds,
              zhist, hist);
  return last();
}
HDK_API int hdk_sdpcg_p(int n3s, int n3, const double* z, double* p, double* pv, const int* p2v, const hdk_pcg* st,
                        int count, int* any, const hdk_defl* d, const hdk_sdefl* ds, const double* w,
                        unsigned long long cond_handle, void* stream) {
  hdk::launch(k_sdpcg_p, dim3(nb(n3)), dim3(256), 0, S(stream), n3s, n3, z, p, pv, p2v, st, count, any, d, ds, w,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle ? 1 : 0);
  return last();
}
HDK_API int hdk_sritz_combine(int n3s, int n3, const double* zhist, const double* coef, int jmax, int k, double* w,
                              void* stream) {
  k_sritz_combine<<<nb(n3), 256, 0, S(stream)>>>(n3s, n3, zhist, coef, jmax, k, w);
  return last();
}

}  // extern "C"
