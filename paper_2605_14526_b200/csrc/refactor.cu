// Device refactorization kernels (refactor.hpp): assembly of A's values for
// a fixed pattern (factor.cpp assemble, same summation order), the
// multifrontal LDL^T one tree level per launch, and D^{-1/2}.  Every
// arithmetic operation is an explicitly rounded intrinsic in the order of the
// host code (factor.cpp assemble; refactor.cpp mf_factor_host), so the device
// values equal the host's bit for bit.
#include <cuda_runtime.h>

#include "../../include/hdk.h"
#include "launch.cuh"

namespace {

constexpr int kPanel = HDK_MF_PANEL;

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// W_e = (2 mu_e + lambda_e + beta_e / h) V_e (factor.cpp assemble)
__global__ void k_asm_weights(int ne, const double* __restrict__ mu, const double* __restrict__ la,
                              const double* __restrict__ beta, const double* __restrict__ vol, double h,
                              double* __restrict__ w) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  w[e] = mul(add(add(mul(2.0, mu[e]), la[e]), __ddiv_rn(beta[e], h)), vol[e]);
}

// out[k] = [diag] inertia m_v + sum over the entry's corner pairs of W_e (g_i . g_j)
__global__ void k_asm_values(int count, const int* __restrict__ off, const int* __restrict__ pair,
                             const int* __restrict__ diag, const double* __restrict__ mass, double inertia,
                             const double* __restrict__ w, const double* __restrict__ g, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  double sum = 0.0;
  if (diag && diag[k] >= 0) sum = add(sum, mul(inertia, mass[diag[k]]));
  for (int q = off[k]; q < off[k + 1]; ++q) {
    const int pr = pair[q];
    const int ei = pr >> 2, j = pr & 3, e = ei >> 2, i = ei & 3;
    const double* ge = g + 12 * (size_t)e;
    const double dot = add(add(mul(ge[3 * i], ge[3 * j]), mul(ge[3 * i + 1], ge[3 * j + 1])), mul(ge[3 * i + 2], ge[3 * j + 2]));
    sum = add(sum, mul(w[e], dot));
  }
  out[k] = sum;
}

__global__ void k_gather_values(int count, const int* __restrict__ from, const double* __restrict__ src,
                                double* __restrict__ dst) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < count) dst[k] = src[from[k]];
}

// One front per CTA: assembly (A entries, children's update blocks in
// order), blocked partial LDL^T of the pivot columns, L and D written out.
template <int kT>
__global__ void __launch_bounds__(kT) k_mf_level(hdk_mf p, int level, const double* __restrict__ aval,
                                                 double* __restrict__ lx, double* __restrict__ d, int* err) {
  const int s = p.level_node[p.level_off[level] + blockIdx.x];
  const int m = p.fm[s], f = p.sfirst[s], piv = p.sfirst[s + 1] - f;
  double* F = p.pool + p.foff[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kT / 32;
  const size_t mm = (size_t)m * m;
  for (size_t q = tid; q < mm; q += kT) F[q] = 0.0;
  __syncthreads();
  for (int k = p.aent_off[s] + tid; k < p.aent_off[s + 1]; k += kT) F[p.aent_dst[k]] = aval[p.aent_src[k]];
  __syncthreads();
  for (int ci = p.child_off[s]; ci < p.child_off[s + 1]; ++ci) {
    const int c = p.child[ci];
    const int mc = p.fm[c], pc = p.sfirst[c + 1] - p.sfirst[c], r = mc - pc;
    const double* U = p.pool + p.foff[c];
    const int* map = p.emap + p.emap_off[c];
    for (int j = warp; j < r; j += nw) {  // column j of the update block, rows j.. by lanes
      const int mj = map[j];
      for (int i = j + lane; i < r; i += 32) {
        double* t = F + map[i] + (size_t)mj * m;
        *t = add(*t, U[(pc + i) + (size_t)(pc + j) * mc]);
      }
    }
    __syncthreads();
  }
  for (int c0 = 0; c0 < piv; c0 += kPanel) {
    const int cb = min(kPanel, piv - c0);
    for (int c = c0; c < c0 + cb; ++c) {
      const double dc = F[c + (size_t)c * m];
      if (!(dc > 0.0)) {  // NotPositiveDefinite (uniform over the CTA)
        if (tid == 0) atomicCAS(err, 0, 8);
        return;
      }
      double* col = F + (size_t)c * m;
      for (int i = c + 1 + tid; i < m; i += kT) col[i] = __ddiv_rn(col[i], dc);
      __syncthreads();
      for (int j = c + 1 + warp; j < c0 + cb; j += nw) {
        const double w = mul(col[j], dc);
        double* cj = F + (size_t)j * m;
        for (int i = j + lane; i < m; i += 32) cj[i] = sub(cj[i], mul(col[i], w));
      }
      __syncthreads();
    }
    for (int j = c0 + cb + warp; j < m; j += nw) {
      double w[kPanel];
#pragma unroll
      for (int c = 0; c < kPanel; ++c)
        w[c] = c < cb ? mul(F[j + (size_t)(c0 + c) * m], F[(c0 + c) + (size_t)(c0 + c) * m]) : 0.0;
      double* cj = F + (size_t)j * m;
      for (int i = j + lane; i < m; i += 32) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < kPanel; ++c)
          if (c < cb) acc = add(acc, mul(F[i + (size_t)(c0 + c) * m], w[c]));
        cj[i] = sub(cj[i], acc);
      }
    }
    __syncthreads();
  }
  for (int c = warp; c < piv; c += nw) {
    const double* col = F + (size_t)c * m;
    if (lane == 0) d[f + c] = col[c];
    const long long base = p.lp[f + c] - (c + 1);
    for (int i = c + 1 + lane; i < m; i += 32) lx[base + i] = col[i];
  }
}

__global__ void k_dis(int n, const double* __restrict__ d, double* __restrict__ dis) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dis[i] = __ddiv_rn(1.0, __dsqrt_rn(d[i]));
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
int last() { return static_cast<int>(cudaGetLastError()); }
int nb(long long n) { return static_cast<int>((n + 255) / 256 > 0 ? (n + 255) / 256 : 1); }

}  // namespace

extern "C" {

HDK_API int hdk_asm_weights(int ne, const double* mu, const double* lambda, const double* beta, const double* vol,
                            double h, double* w, void* stream) {
  k_asm_weights<<<nb(ne), 256, 0, S(stream)>>>(ne, mu, lambda, beta, vol, h, w);
  return last();
}

HDK_API int hdk_asm_values(int count, const int* off, const int* pair, const int* diag, const double* mass,
                           double inertia, const double* w, const double* g, double* out, void* stream) {
  if (count <= 0) return 0;
  k_asm_values<<<nb(count), 256, 0, S(stream)>>>(count, off, pair, diag, mass, inertia, w, g, out);
  return last();
}

HDK_API int hdk_gather_values(int count, const int* from, const double* src, double* dst, void* stream) {
  if (count <= 0) return 0;
  k_gather_values<<<nb(count), 256, 0, S(stream)>>>(count, from, src, dst);
  return last();
}

HDK_API int hdk_mf_factor(const hdk_mf* p, const double* aval, double* lx, double* d, double* dis, int* err,
                          void* stream) {
  for (int L = 0; L < p->nlevels; ++L) {  // wide CTAs where the fronts are large (the top levels)
    const int fronts = p->h_level_off[L + 1] - p->h_level_off[L];
    if (p->h_level_maxm[L] >= 192) k_mf_level<1024><<<fronts, 1024, 0, S(stream)>>>(*p, L, aval, lx, d, err);
    else k_mf_level<256><<<fronts, 256, 0, S(stream)>>>(*p, L, aval, lx, d, err);
  }
  k_dis<<<nb(p->n), 256, 0, S(stream)>>>(p->n, d, dis);
  return last();
}

}  // extern "C"
