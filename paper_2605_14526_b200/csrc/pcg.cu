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

constexpr int kSRB = HDK_SEG_RB;

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
  hdk::pdl_wait();
  hdk::pdl_trigger();
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
  const hdk_pcg& c = st[i / n3s];
  if (c.cond == 0) return;
  const double v = z[i] + c.beta * p[i];
  p[i] = v;
  const int row = i / 3;
  pv[3 * (size_t)__ldg(p2v + row) + (i - 3 * row)] = v;
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
__global__ void __launch_bounds__(kT) k_cpcg_apply(hdk_vtx x, hdk_csr A, int n3, const double* __restrict__ ef,
                                                   size_t ef_stride, const double* __restrict__ p,
                                                   double* __restrict__ q, double* partial, size_t pstride,
                                                   unsigned int* tickets, hdk_pcg* sts) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int c = blockIdx.y;
  hdk_pcg* st = sts + c;
  if (st->cond == 0) return;
  const double* efc = ef + c * ef_stride;
  const double* pc = p + (size_t)c * n3;
  double* qc = q + (size_t)c * n3;
  const int sub = threadIdx.x & 7;
  const int row = blockIdx.x * (kT / 8) + (threadIdx.x >> 3);
  const bool live = row < x.n;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0;
  const int e = live ? __ldg(x.pinc_off + row + 1) : 0;
  for (int j = (live ? __ldg(x.pinc_off + row) : 0) + sub; j < e; j += 8) {
    const double* f = efc + 3 * (size_t)j;
    c0 += __ldg(f);
    c1 += __ldg(f + 1);
    c2 += __ldg(f + 2);
  }
  const int ke = live ? __ldg(A.off + row + 1) : 0;
  for (int k = (live ? __ldg(A.off + row) : 0) + sub; k < ke; k += 8) {
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
  hdk::launch(k_cpcg_apply, dim3(nbx > 0 ? nbx : 1, columns), dim3(kT), 0, S(stream), *x, *a, 3 * x->n, ef_sorted,
              ef_stride, p, q, partial, pstride, tickets, st);
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
