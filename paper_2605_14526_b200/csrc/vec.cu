// Vertex- and DoF-parallel kernels of the PD loop: fixed-order element-force
// gathers (the serial scatters of pd_rhs/damping_rhs, forward.cpp:96-138),
// Type-II Anderson mixing with its small coefficient solve (forward.cpp:17-51),
// the dual gate (forward.cpp:140-146), the trust-region ratio
// (backward.cpp:75-108) and the vertex part of route_gradients
// (backward.cpp:296-356).
//
// Reductions: every reducing kernel runs a fixed grid of HDK_RED_BLOCKS x 256
// threads with grid-stride loops and writes one partial per block; a
// single-block kernel folds the partials in a fixed tree.  Results are
// bitwise reproducible run to run (no atomics on doubles).
#include <cuda_runtime.h>

#include <cmath>

#include "../../include/hdk.h"
#include "launch.cuh"

namespace {

constexpr int kT = 256;

template <int NQ>
__device__ __forceinline__ void block_partials(double (&v)[NQ], double* partial) {
  __shared__ double sm[kT / 32][NQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double x = v[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) sm[warp][q] = x;
  }
  __syncthreads();
  if (threadIdx.x < NQ) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) s += sm[w][threadIdx.x];
    partial[blockIdx.x * HDK_RED_Q + threadIdx.x] = s;
  }
}

// Single-block fold of partial slots [0, nq) over all blocks (fixed order):
// warp w folds slots w, w + nwarps, ...; each lane issues all of its loads
// before adding (no latency chain), then a fixed shuffle tree.  out must be
// shared memory; the caller syncs after.
constexpr int kFoldPerLane = (HDK_RED_BLOCKS + 31) / 32;
__device__ __forceinline__ void fold_all(const double* __restrict__ partial, int nq, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll 1
  for (int q = warp; q < nq; q += nw) {
    double v[kFoldPerLane];
#pragma unroll
    for (int i = 0; i < kFoldPerLane; ++i) {
      const int b = lane + 32 * i;
      v[i] = b < HDK_RED_BLOCKS ? __ldcg(partial + b * HDK_RED_Q + q) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kFoldPerLane; ++i) s += v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[q] = s;
  }
}

// Fixed-order sum of the element forces incident to vertex v (ascending
// element order = the reference's serial scatter order).
__device__ __forceinline__ void gather_vtx(const hdk_vtx& x, const double* __restrict__ ef, int v, double& s0,
                                           double& s1, double& s2) {
  s0 = s1 = s2 = 0.0;
  const int e = x.inc_off[v + 1];
#pragma unroll 4
  for (int j = x.inc_off[v]; j < e; ++j) {
    const double* p = ef + 3 * (size_t)__ldg(x.inc + j);
    s0 += __ldg(p);
    s1 += __ldg(p + 1);
    s2 += __ldg(p + 2);
  }
}

__global__ void k_free_fall(hdk_vtx x, const double* q, const double* v, const double* f, double h, int hv,
                            double ax, double ay, double az, double hk, double hd, double* qt, double* qc) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * x.nv) return;
  const int vtx = i / 3, a = i - 3 * vtx;
  double force = f[i];
  if (vtx == hv) {
    const double anc = a == 0 ? ax : a == 1 ? ay : az;
    force += -hk * (q[i] - anc) - hd * v[i];
  }
  const double t = q[i] + h * v[i] + (h * h) * (force / x.mass[vtx]);
  qt[i] = t;
  qc[i] = x.v2p[vtx] < 0 ? q[i] : t;
}

__global__ void k_gather(hdk_vtx x, const double* ef, double cm, const double* base, const double* add, double* out) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= x.nv) return;
  double g[3] = {0.0, 0.0, 0.0};
  if (ef) gather_vtx(x, ef, v, g[0], g[1], g[2]);
  for (int a = 0; a < 3; ++a) {
    double s = cm * x.mass[v] * base[3 * v + a];
    if (add) s += add[3 * v + a];
    s += g[a];
    out[3 * v + a] = s;
  }
}

__global__ void __launch_bounds__(kT) k_gather_rhs(hdk_vtx x, const double* __restrict__ ef, double inv_h2,
                                                   const double* __restrict__ qt, const double* __restrict__ damp,
                                                   const double* __restrict__ fixc, double* bprev, double* rhs,
                                                   double* partial) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  double acc[2] = {0.0, 0.0};
  for (int v = blockIdx.x * kT + threadIdx.x; v < x.nv; v += HDK_RED_BLOCKS * kT) {
    const int p = x.v2p[v];
    const double m = x.mass[v];
    double g[3];
    gather_vtx(x, ef, v, g[0], g[1], g[2]);
    for (int a = 0; a < 3; ++a) {
      const size_t i = 3 * (size_t)v + a;
      double b = m * qt[i] * inv_h2;  // M q~ / h^2 (forward.cpp:99)
      b += g[a];                      // + sum_e V G^T (w p*)
      b += damp[i];                   // + damping_rhs
      const double d = b - bprev[i];
      acc[0] += d * d;
      acc[1] += b * b;
      bprev[i] = b;
      if (p >= 0) rhs[3 * (size_t)p + a] = b - (fixc ? fixc[3 * (size_t)p + a] : 0.0);
    }
  }
  block_partials<2>(acc, partial);
}

// rhs[p] = base[v] + sum of incident element forces, v = p2v[p].  Eight lanes
// per vertex split the incidence list (fixed lane assignment) and fold it
// with a fixed shuffle tree.
__global__ void k_gather_perm(hdk_vtx x, const double* __restrict__ base, const double* __restrict__ ef,
                              double* __restrict__ rhs) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = gid >> 3, sub = gid & 7;
  const bool live = p < x.n;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  int v = 0;
  if (live) {
    v = x.p2v[p];
    if (ef) {
      const int e = x.inc_off[v + 1];
#pragma unroll 4
      for (int j = x.inc_off[v] + sub; j < e; j += 8) {
        const double* q = ef + 3 * (size_t)__ldg(x.inc + j);
        s0 += __ldg(q);
        s1 += __ldg(q + 1);
        s2 += __ldg(q + 2);
      }
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (live && sub == 0) {
    rhs[3 * (size_t)p] = base[3 * (size_t)v] + s0;
    rhs[3 * (size_t)p + 1] = base[3 * (size_t)v + 1] + s1;
    rhs[3 * (size_t)p + 2] = base[3 * (size_t)v + 2] + s2;
  }
}

__global__ void k_fixed_coupling(hdk_csr c, const int* fixed, const double* q, double* out) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= c.rows) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int k = c.off[p]; k < c.off[p + 1]; ++k) {
    const double w = c.val[k];
    const int v = fixed[c.col[k]];
    s0 += w * q[3 * (size_t)v];
    s1 += w * q[3 * (size_t)v + 1];
    s2 += w * q[3 * (size_t)v + 2];
  }
  out[3 * (size_t)p] = s0;
  out[3 * (size_t)p + 1] = s1;
  out[3 * (size_t)p + 2] = s2;
}

// ---- Anderson mixing ---------------------------------------------------------
__global__ void __launch_bounds__(kT) k_aa_dots(hdk_vtx x, const hdk_ctl* ctl, const double* __restrict__ qhat,
                                                const double* __restrict__ qcur, double* last_q, double* last_g,
                                                double* dq, double* dg, double* partial) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const size_t n3 = 3 * (size_t)x.nv;
  const int m = ctl->window, c = ctl->count, h = ctl->head;
  const bool push = ctl->has_last != 0;
  int ns = 0, c2 = c, h2 = h;
  if (push) {
    ns = c < m ? (h + c) % m : h;
    c2 = c < m ? c + 1 : m;
    h2 = c < m ? h : (h + 1) % m;
  }
  double acc[2 * HDK_AA_MAX + 2];
#pragma unroll
  for (int q = 0; q < 2 * HDK_AA_MAX + 2; ++q) acc[q] = 0.0;
  for (size_t i = blockIdx.x * kT + threadIdx.x; i < n3; i += (size_t)HDK_RED_BLOCKS * kT) {
    const double qc = qcur[i], th = qhat[i];
    const double g = th - qc;
    acc[2 * HDK_AA_MAX] += g * g;
    acc[2 * HDK_AA_MAX + 1] += th * th;
    if (push) {
      const double dqn = qc - last_q[i];
      const double dgn = g - last_g[i];
      dq[ns * n3 + i] = dqn;
      dg[ns * n3 + i] = dgn;
#pragma unroll
      for (int j = 0; j < HDK_AA_MAX; ++j) {
        if (j < c2) {
          const int ph = (h2 + j) % m;
          const double dgj = ph == ns ? dgn : dg[ph * n3 + i];
          acc[j] += dgn * dgj;
          acc[HDK_AA_MAX + j] += dgj * g;
        }
      }
    }
    last_q[i] = qc;
    last_g[i] = g;
  }
  block_partials<2 * HDK_AA_MAX + 2>(acc, partial);
}

// Anderson coefficient solve (forward.cpp:31-47): M gamma = DG^T g with
// M = DG^T DG + 1e-6 |DG|_F^2 / window I, by LDL^T with Eigen::LDLT's
// diagonal pivoting (left-looking, pivots chosen on the untouched diagonal).
// One warp: lane 0 does the short serial bookkeeping, the factorization runs
// row-parallel over lanes; everything lives in shared memory.
// Runs on one whole block of kT threads: inside k_aa_solve, or as the tail of
// k_aa_dots_fused in whichever block finishes last.  mode 1 also sets the
// adjoint loop's WHILE condition (the former k_bb_cond) when a graph handle
// is given.
constexpr int kSolveT = kT;  // 8 warps fold the 18 partial sums
__device__ __noinline__ void aa_solve_block(hdk_ctl* gctl, const double* partial, int mode,
                                            cudaGraphConditionalHandle handle, int use_handle) {
  __shared__ double s[2 * HDK_AA_MAX + 2];
  __shared__ hdk_ctl c;  // shared-memory copy of the control block
  __shared__ double A[HDK_AA_MAX][HDK_AA_MAX + 1], L[HDK_AA_MAX][HDK_AA_MAX + 1], d[HDK_AA_MAX], y[HDK_AA_MAX];
  __shared__ int perm[HDK_AA_MAX], solve_n, ok;
  {
    const int* src = reinterpret_cast<const int*>(gctl);
    int* dst = reinterpret_cast<int*>(&c);
    #pragma unroll 1
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(hdk_ctl) / 4); i += blockDim.x) dst[i] = src[i];
  }
  fold_all(partial, 2 * HDK_AA_MAX + 2, s);
  __syncthreads();
  if (threadIdx.x >= 32) goto writeback;
  {
    const int lane = threadIdx.x;
    if (lane == 0) {
      solve_n = 0;
      bool skip = false;
      if (mode == 1) {  // adjoint backbone: convergence test before mixing (backward.cpp:191-193)
        c.iterations += 1;
        const double diff = sqrt(s[2 * HDK_AA_MAX]);
        const double base = fmax(sqrt(s[2 * HDK_AA_MAX + 1]), 1e-30);
        c.k += 1;
        if (diff <= c.tol * base) {
          c.done = 1;
          c.mixed = 0;
          skip = true;
        } else if (c.k >= c.k_max && c.err == 0) {
          c.err = 10;  // AdjointDiverged (cap)
        }
      }
      if (!skip) {
        const int m = c.window;
        if (c.has_last) {
          const int n0 = c.count;
          if (n0 < m) {
            c.count = n0 + 1;
          } else {
            c.head = (c.head + 1) % m;
            #pragma unroll 1
            for (int i = 0; i + 1 < m; ++i)
              #pragma unroll 1
              for (int j = 0; j + 1 < m; ++j) c.gram[i * HDK_AA_MAX + j] = c.gram[(i + 1) * HDK_AA_MAX + (j + 1)];
          }
          const int n1 = c.count, j = n1 - 1;
          #pragma unroll 1
          for (int l = 0; l < n1; ++l) c.gram[j * HDK_AA_MAX + l] = c.gram[l * HDK_AA_MAX + j] = s[l];
        }
        c.has_last = 1;
        c.mixed = 0;
        const int n = c.count;
        double fro2 = 0.0;
        #pragma unroll 1
        for (int j = 0; j < n; ++j) fro2 += c.gram[j * HDK_AA_MAX + j];
        if (n > 0 && fro2 > 0.0) {
          solve_n = n;
          // pivot order: Eigen picks the largest |diagonal| among the remaining
          // (untouched) diagonal entries, swapping it into place
          double dg[HDK_AA_MAX];
          #pragma unroll 1
          for (int i = 0; i < n; ++i) {
            perm[i] = i;
            dg[i] = c.gram[i * HDK_AA_MAX + i] + 1e-6 * fro2 / m;
          }
          #pragma unroll 1
          for (int k = 0; k < n; ++k) {
            int piv = k;
            double best = fabs(dg[k]);
            #pragma unroll 1
            for (int i = k + 1; i < n; ++i)
              if (fabs(dg[i]) > best) { best = fabs(dg[i]); piv = i; }
            const int tp = perm[k]; perm[k] = perm[piv]; perm[piv] = tp;
            const double td = dg[k]; dg[k] = dg[piv]; dg[piv] = td;
          }
          y[0] = 1e-6 * fro2 / m;  // ridge, broadcast below
        }
      }
    }
    __syncwarp();
    const int n = solve_n;
    if (n > 0) {
      const double ridge = y[0];
      __syncwarp();
      // permuted matrix, rows over lanes
      #pragma unroll 1
      for (int e = lane; e < n * n; e += 32) {
        const int i = e / n, j = e % n;
        A[i][j] = c.gram[perm[i] * HDK_AA_MAX + perm[j]] + (perm[i] == perm[j] ? ridge : 0.0);
      }
      __syncwarp();
      if (lane == 0) ok = 1;
      __syncwarp();
      #pragma unroll 1
      for (int k = 0; k < n; ++k) {
        if (lane == k) {
          double dk = A[k][k];
          #pragma unroll 1
          for (int j = 0; j < k; ++j) dk -= L[k][j] * L[k][j] * d[j];
          d[k] = dk;
          if (!(fabs(dk) > 2.2250738585072014e-308)) ok = 0;
        }
        __syncwarp();
        if (lane > k && lane < n) {
          double v = A[lane][k];
          #pragma unroll 1
          for (int j = 0; j < k; ++j) v -= L[lane][j] * L[k][j] * d[j];
          L[lane][k] = v / d[k];
        }
        __syncwarp();
      }
      if (lane == 0) {
        double gam[HDK_AA_MAX];
        bool good = ok != 0;
        if (good) {
          #pragma unroll 1
          for (int i = 0; i < n; ++i) y[i] = s[HDK_AA_MAX + perm[i]];
          #pragma unroll 1
          for (int i = 0; i < n; ++i)
            #pragma unroll 1
            for (int j = 0; j < i; ++j) y[i] -= L[i][j] * y[j];
          #pragma unroll 1
          for (int i = 0; i < n; ++i) y[i] /= d[i];
          #pragma unroll 1
          for (int i = n - 1; i >= 0; --i)
            #pragma unroll 1
            for (int j = i + 1; j < n; ++j) y[i] -= L[j][i] * y[j];
          #pragma unroll 1
          for (int i = 0; i < n; ++i) gam[perm[i]] = y[i];
          #pragma unroll 1
          for (int i = 0; i < n; ++i) good = good && isfinite(gam[i]);
        }
        double gn = 0.0;
        if (good)
          #pragma unroll 1
          for (int i = 0; i < n; ++i) gn += gam[i] * gam[i];
        if (!good || !(sqrt(gn) <= c.guard)) {  // guard: discard history (forward.cpp:43-47)
          c.count = 0;
          c.head = 0;
          c.has_last = 0;
        } else {
          #pragma unroll 1
          for (int i = 0; i < n; ++i) c.gamma[i] = gam[i];
          c.mixed = 1;
        }
      }
    }
  }
writeback:
  __syncthreads();
  if (mode == 1 && threadIdx.x == 0) {  // adjoint loop condition (done / error)
    c.cond = (!c.done && c.err == 0) ? 1 : 0;
    if (use_handle) cudaGraphSetConditional(handle, c.cond);
  }
  __syncthreads();
  {
    const int* src = reinterpret_cast<const int*>(&c);
    int* dst = reinterpret_cast<int*>(gctl);
    #pragma unroll 1
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(hdk_ctl) / 4); i += blockDim.x) dst[i] = src[i];
  }
}

__global__ void __launch_bounds__(kSolveT) k_aa_solve(hdk_ctl* gctl, const double* partial, int mode) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  aa_solve_block(gctl, partial, mode, 0, 0);
}

// Fused tail of one PD / adjoint iteration after the solve's column pass:
//   * x-fold (the former k_xreduce): qhat at free vertex v is the fixed-order
//     sum of the pass-2 tile partials of column p = v2p[v] — same terms, same
//     order, so bitwise what k_xreduce scattered; fixed rows keep qhat;
//   * the Anderson history update and dot partials (k_aa_dots);
//   * the coefficient solve (k_aa_solve) in the block that finishes last
//     (threadfence + ticket), and in mode 1 the loop condition.
// One launch instead of four.
__global__ void __launch_bounds__(kT) k_aa_dots_fused(hdk_vtx x, hdk_factor f, int g2, hdk_ctl* ctl,
                                                      double* __restrict__ qhat, const double* __restrict__ qcur,
                                                      double* last_q, double* last_g, double* dq, double* dg,
                                                      double* partial, unsigned int* ticket, int mode,
                                                      cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const size_t n3 = 3 * (size_t)x.nv;
  const int m = ctl->window, c = ctl->count, h = ctl->head;
  const bool push = ctl->has_last != 0;
  int ns = 0, c2 = c, h2 = h;
  if (push) {
    ns = c < m ? (h + c) % m : h;
    c2 = c < m ? c + 1 : m;
    h2 = c < m ? h : (h + 1) % m;
  }
  double acc[2 * HDK_AA_MAX + 2];
#pragma unroll
  for (int q = 0; q < 2 * HDK_AA_MAX + 2; ++q) acc[q] = 0.0;
  for (size_t i = blockIdx.x * kT + threadIdx.x; i < n3; i += (size_t)HDK_RED_BLOCKS * kT) {
    const int v = static_cast<int>(i / 3), a = static_cast<int>(i - 3 * (size_t)v);
    const int p = __ldg(x.v2p + v);
    double th;
    if (p >= 0) {
      const int t = p / 256, cl = p - 256 * t;
      const int b0 = f.tile_cta2 ? __ldg(f.tile_cta2 + 2 * t) : 0;
      const int b1 = f.tile_cta2 ? __ldg(f.tile_cta2 + 2 * t + 1) : -1;
      th = 0.0;
      for (int b = b0; b <= b1; ++b) th += __ldcg(f.part2 + 3 * ((size_t)(t + b) * 256 + cl) + a);
      qhat[i] = th;
    } else {
      th = qhat[i];
    }
    const double qc = qcur[i];
    const double g = th - qc;
    acc[2 * HDK_AA_MAX] += g * g;
    acc[2 * HDK_AA_MAX + 1] += th * th;
    if (push) {
      const double dqn = qc - last_q[i];
      const double dgn = g - last_g[i];
      dq[ns * n3 + i] = dqn;
      dg[ns * n3 + i] = dgn;
#pragma unroll
      for (int j = 0; j < HDK_AA_MAX; ++j) {
        if (j < c2) {
          const int ph = (h2 + j) % m;
          const double dgj = ph == ns ? dgn : dg[ph * n3 + i];
          acc[j] += dgn * dgj;
          acc[HDK_AA_MAX + j] += dgj * g;
        }
      }
    }
    last_q[i] = qc;
    last_g[i] = g;
  }
  block_partials<2 * HDK_AA_MAX + 2>(acc, partial);
  // last block folds every partial and runs the coefficient solve
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(ticket, 1u);
    is_last = t == gridDim.x - 1;
    if (is_last) *ticket = 0u;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  aa_solve_block(ctl, partial, mode, handle, use_handle);
}

__global__ void __launch_bounds__(kT) k_aa_mix(hdk_vtx x, hdk_ctl* ctl, const double* __restrict__ qhat, double* qcur,
                                               double* qprev, const double* __restrict__ qpin,
                                               const double* __restrict__ dq, const double* __restrict__ dg,
                                               double* partial, int mode) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const size_t n3 = 3 * (size_t)x.nv;
  const bool done = mode == 1 && ctl->done;
  const int mixed = ctl->mixed, c = ctl->count, h = ctl->head, m = ctl->window;
  double gam[HDK_AA_MAX];
#pragma unroll
  for (int j = 0; j < HDK_AA_MAX; ++j) gam[j] = j < c ? ctl->gamma[j] : 0.0;
  double acc[2] = {0.0, 0.0};
  bool finite = true;
  for (size_t i = blockIdx.x * kT + threadIdx.x; i < n3; i += (size_t)HDK_RED_BLOCKS * kT) {
    const double qc = qcur[i], th = qhat[i];
    double out = qc + (th - qc);
    if (done) {
      out = th;
    } else if (mixed) {
#pragma unroll
      for (int j = 0; j < HDK_AA_MAX; ++j)
        if (j < c) {
          const int ph = (h + j) % m;
          out -= gam[j] * (dq[ph * n3 + i] + dg[ph * n3 + i]);
        }
    }
    if (mode == 0) {
      if (x.v2p[i / 3] < 0) out = qpin[i];
      const double d = out - qc;
      acc[0] += d * d;
      acc[1] += qc * qc;
      qprev[i] = qc;
    } else {
      finite = finite && isfinite(out);
    }
    qcur[i] = out;
  }
  if (mode == 0) block_partials<2>(acc, partial);
  else if (!finite) atomicCAS(&ctl->err, 0, 10);
}

__global__ void __launch_bounds__(kT) k_gate(hdk_ctl* ctl, const double* pb, const double* pq,
                                             cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  __shared__ double sb[2], sq[2];
  fold_all(pb, 2, sb);
  fold_all(pq, 2, sq);
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double db = sb[0], bb = sb[1], dq = sq[0], qq = sq[1];
  const int k = ctl->k;
  const double er = ctl->eps_rel, ea = ctl->eps_abs;
  const bool gate = k >= 1 && sqrt(dq) <= er * sqrt(qq) + ea && sqrt(db) <= er * sqrt(bb) + ea;
  ctl->k = k + 1;
  ctl->iterations = k + 1;
  if (gate) ctl->converged = 1;
  const int cont = (!gate && k + 1 < ctl->k_max && ctl->err == 0) ? 1 : 0;
  ctl->cond = cont;
  if (use_handle) cudaGraphSetConditional(handle, cont);
}

__global__ void k_bb_cond(hdk_ctl* ctl, cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int cont = (!ctl->done && ctl->err == 0) ? 1 : 0;
  ctl->cond = cont;
  if (use_handle) cudaGraphSetConditional(handle, cont);
}

// ---- trust-region ratio --------------------------------------------------------
__global__ void k_tr_dq(hdk_vtx x, const double* qs, const double* qp, double* dq) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= x.n) return;
  const int v = x.p2v[p];
  for (int a = 0; a < 3; ++a) dq[3 * (size_t)p + a] = qs[3 * (size_t)v + a] - qp[3 * (size_t)v + a];
}

__global__ void __launch_bounds__(kT) k_tr_spmv(hdk_csr A, const double* __restrict__ dq, double* partial) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  double acc[1] = {0.0};
  for (int p = blockIdx.x * kT + threadIdx.x; p < A.rows; p += HDK_RED_BLOCKS * kT) {
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    for (int k = A.off[p]; k < A.off[p + 1]; ++k) {
      const double w = A.val[k];
      const double* d = dq + 3 * (size_t)A.col[k];
      y0 += w * d[0];
      y1 += w * d[1];
      y2 += w * d[2];
    }
    const double* d = dq + 3 * (size_t)p;
    acc[0] += d[0] * y0 + d[1] * y1 + d[2] * y2;
  }
  block_partials<1>(acc, partial);
}

__global__ void __launch_bounds__(kT) k_tr_partials(hdk_vtx x, int ne, const double* ep, const double* es,
                                                    const double* qp, const double* qs, const double* qt,
                                                    double* partial) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int n = max(ne, x.nv);
  for (int i = blockIdx.x * kT + threadIdx.x; i < n; i += HDK_RED_BLOCKS * kT) {
    if (i < ne) {
      acc[0] += ep[i];
      acc[1] += es[i];
    }
    if (i < x.nv && x.v2p[i] >= 0) {
      const double m = x.mass[i];
      for (int a = 0; a < 3; ++a) {
        const size_t j = 3 * (size_t)i + a;
        const double d0 = qp[j] - qt[j], d1 = qs[j] - qt[j];
        acc[2] += d0 * m * d0;
        acc[3] += d1 * m * d1;
      }
    }
  }
  block_partials<4>(acc, partial);
}

__global__ void __launch_bounds__(kT) k_tr_final(hdk_ctl* ctl, const double* pm, const double* pe, double inv_h2) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  __shared__ double sm_[1], se[4];
  fold_all(pm, 1, sm_);
  fold_all(pe, 4, se);
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double model_raw = sm_[0], e_prev = se[0], e_star = se[1], i_prev = se[2], i_star = se[3];
  const double model = 0.5 * fabs(model_raw);
  double rho = 1.0;
  if (model >= 1e-12) {
    if (ctl->bad != 0) {
      rho = INFINITY;
    } else {
      const double phi_prev = 0.5 * inv_h2 * i_prev + e_prev;
      const double phi_star = 0.5 * inv_h2 * i_star + e_star;
      rho = (phi_prev - phi_star) / model;
    }
  }
  ctl->model = model;
  ctl->rho = rho;
  ctl->tau = fabs(rho - 1.0) <= ctl->eps_tr ? 0.5 : 1.0;
}

// ---- gradient routing ------------------------------------------------------------
__global__ void k_route_vtx(hdk_vtx x, const double* mu, const double* efd, const double* bmu, const double* qbar,
                            const double* vbar, const double* coup, double h, double alpha, int hv, double hk,
                            double hd, double* dq_t, double* dv_t, double* df_acc) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= x.nv) return;
  const double m = x.mass[v];
  const bool fixed = x.v2p[v] < 0;
  double g[3] = {0.0, 0.0, 0.0};
  if (efd) gather_vtx(x, efd, v, g[0], g[1], g[2]);
  for (int a = 0; a < 3; ++a) {
    const size_t i = 3 * (size_t)v + a;
    const double u = mu[i];
    df_acc[i] += u;                            // dL/df_ext = mu (backward.cpp:303)
    double dv = m * u / h;                     // M mu / h
    double damp = 0.0;
    if (alpha > 0) damp = (alpha / h) * (m * u);
    if (efd) damp += g[a];
    double dq = m * u / (h * h) + damp;        // M mu / h^2 + damping_rhs(mu)
    if (v == hv) {
      dv += -hd * u;
      dq += -hk * u;
    }
    if (!fixed) {
      dq -= vbar[i] / h;
    } else {
      dq += qbar[i];
      if (bmu) dq += bmu[i];
      if (coup) dq -= coup[i];
    }
    dq_t[i] = dq;
    dv_t[i] = dv;
  }
}

__global__ void k_fixed_coupling_t(hdk_csr c, const int* fixed, const int* p2v, const double* mu, double* coup) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= c.rows) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int j = c.off[k]; j < c.off[k + 1]; ++j) {
    const double w = c.val[j];
    const int v = p2v[c.col[j]];
    s0 += w * mu[3 * (size_t)v];
    s1 += w * mu[3 * (size_t)v + 1];
    s2 += w * mu[3 * (size_t)v + 2];
  }
  const int v = fixed[k];
  coup[3 * (size_t)v] = s0;
  coup[3 * (size_t)v + 1] = s1;
  coup[3 * (size_t)v + 2] = s2;
}

__global__ void k_axpby(int n, double a, const double* x, double b, const double* z, double* y) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = a * x[i];
  if (z) s += b * z[i];
  y[i] = s;
}

__global__ void k_velocity(int n, const double* qs, const double* qt, double h, double* vs) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) vs[i] = (qs[i] - qt[i]) / h;
}

__global__ void k_ctl_init(hdk_ctl* c, int window, double guard, int k_max, double er, double ea, double tol,
                           double eps_tr, int it0) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  c->k = 0; c->k_max = k_max; c->iterations = it0; c->converged = 0;
  c->err = 0; c->done = 0; c->bad = 0; c->cond = 1;
  c->window = window < 1 ? 1 : window; c->count = 0; c->head = 0; c->has_last = 0; c->mixed = 0;
  c->eps_rel = er; c->eps_abs = ea; c->guard = guard; c->tol = tol;
  c->tau = 1.0; c->rho = 1.0; c->model = 0.0; c->eps_tr = eps_tr;
  for (int i = 0; i < HDK_AA_MAX; ++i) c->gamma[i] = 0.0;
  for (int i = 0; i < HDK_AA_MAX * HDK_AA_MAX; ++i) c->gram[i] = 0.0;
}

// Resets the loop / Anderson fields only (keeps tau, rho, bad, err).
__global__ void k_aa_reset(hdk_ctl* c, int window, double guard, int k_max, double tol) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  c->k = 0; c->k_max = k_max; c->iterations = 0; c->converged = 0; c->done = 0; c->cond = 1;
  c->window = window < 1 ? 1 : window; c->count = 0; c->head = 0; c->has_last = 0; c->mixed = 0;
  c->guard = guard; c->tol = tol;
}

__global__ void k_commit(int n, const hdk_ctl* ctl, const double* qs, double h, double* q, double* v) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || ctl->err != 0) return;
  const double s = qs[i];
  v[i] = (s - q[i]) / h;
  q[i] = s;
}

inline int nb(long long n) { return static_cast<int>((n + 255) / 256); }
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
inline int last() { return static_cast<int>(cudaGetLastError()); }

}  // namespace

extern "C" {

HDK_API int hdk_free_fall(const hdk_vtx* x, const double* q, const double* v, const double* f_ext, double h,
                          int hook_vertex, const double* hook, double* q_tilde, double* q_cur, void* stream) {
  const double z[5] = {0, 0, 0, 0, 0};
  const double* hp = hook ? hook : z;
  hdk::launch(k_free_fall, dim3(nb(3LL * x->nv)), dim3(256), 0, S(stream), *x, q, v, f_ext, h, hook ? hook_vertex : -1, hp[0], hp[1], hp[2],
                                                       hp[3], hp[4], q_tilde, q_cur);
  return last();
}

HDK_API int hdk_gather(const hdk_vtx* x, const double* ef, double cm, const double* base, const double* add, double* out,
                       void* stream) {
  hdk::launch(k_gather, dim3(nb(x->nv)), dim3(256), 0, S(stream), *x, ef, cm, base, add, out);
  return last();
}

HDK_API int hdk_gather_rhs(const hdk_vtx* x, const double* ef, double inv_h2, const double* q_tilde, const double* damp,
                           const double* fixcoup, double* b_prev, double* rhs_perm, double* partial, void* stream) {
  hdk::launch(k_gather_rhs, dim3(HDK_RED_BLOCKS), dim3(kT), 0, S(stream), *x, ef, inv_h2, q_tilde, damp, fixcoup, b_prev, rhs_perm, partial);
  return last();
}

HDK_API int hdk_gather_perm(const hdk_vtx* x, const double* base, const double* ef, double* rhs_perm, void* stream) {
  hdk::launch(k_gather_perm, dim3(nb(8LL * x->n)), dim3(256), 0, S(stream), *x, base, ef, rhs_perm);
  return last();
}

HDK_API int hdk_fixed_coupling(const hdk_csr* a_fd, const int* fixed, const double* q, double* fixcoup, void* stream) {
  hdk::launch(k_fixed_coupling, dim3(nb(a_fd->rows)), dim3(256), 0, S(stream), *a_fd, fixed, q, fixcoup);
  return last();
}

HDK_API int hdk_aa_dots(const hdk_vtx* x, hdk_ctl* ctl, const double* qhat, const double* qcur, double* last_q,
                        double* last_g, double* dq, double* dg, double* partial, void* stream) {
  hdk::launch(k_aa_dots, dim3(HDK_RED_BLOCKS), dim3(kT), 0, S(stream), *x, ctl, qhat, qcur, last_q, last_g, dq, dg, partial);
  return last();
}

HDK_API int hdk_aa_solve(hdk_ctl* ctl, const double* partial, int mode, void* stream) {
  hdk::launch(k_aa_solve, dim3(1), dim3(kSolveT), 0, S(stream), ctl, partial, mode);
  return last();
}

HDK_API int hdk_aa_dots_fused(const hdk_vtx* x, const hdk_factor* f, hdk_ctl* ctl, double* qhat, const double* qcur,
                              double* last_q, double* last_g, double* dq, double* dg, double* partial,
                              unsigned int* ticket, int mode, unsigned long long cond_handle, void* stream) {
  int g1 = 0, g2 = 0;
  hdk_solve_grids(f, &g1, &g2);
  if (!f->tile_cta2 || g2 != f->grid2) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_aa_dots_fused, dim3(HDK_RED_BLOCKS), dim3(kT), 0, S(stream), *x, *f, g2, ctl, qhat, qcur, last_q,
              last_g, dq, dg, partial, ticket, mode, static_cast<cudaGraphConditionalHandle>(cond_handle),
              cond_handle != 0ULL ? 1 : 0);
  return last();
}

HDK_API int hdk_aa_mix(const hdk_vtx* x, hdk_ctl* ctl, const double* qhat, double* qcur, double* qprev,
                       const double* qpin, const double* dq, const double* dg, double* partial, int mode,
                       void* stream) {
  hdk::launch(k_aa_mix, dim3(HDK_RED_BLOCKS), dim3(kT), 0, S(stream), *x, ctl, qhat, qcur, qprev, qpin, dq, dg, partial, mode);
  return last();
}

HDK_API int hdk_gate(hdk_ctl* ctl, const double* partial_b, const double* partial_q, unsigned long long cond_handle,
                     void* stream) {
  hdk::launch(k_gate, dim3(1), dim3(kT), 0, S(stream), ctl, partial_b, partial_q, static_cast<cudaGraphConditionalHandle>(cond_handle),
                                   cond_handle != 0ULL);
  return last();
}

HDK_API int hdk_backbone_cond(hdk_ctl* ctl, unsigned long long cond_handle, void* stream) {
  hdk::launch(k_bb_cond, dim3(1), dim3(1), 0, S(stream), ctl, static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle != 0ULL);
  return last();
}

HDK_API int hdk_tr_model(const hdk_vtx* x, const hdk_csr* a_ff, const double* q_star, const double* q_prev,
                         double* dq_perm, double* partial, void* stream) {
  hdk::launch(k_tr_dq, dim3(nb(x->n)), dim3(256), 0, S(stream), *x, q_star, q_prev, dq_perm);
  hdk::launch(k_tr_spmv, dim3(HDK_RED_BLOCKS), dim3(kT), 0, S(stream), *a_ff, dq_perm, partial);
  return last();
}

HDK_API int hdk_tr_select(const hdk_vtx* x, int ne, const double* e_prev, const double* e_star, const double* q_prev,
                          const double* q_star, const double* q_tilde, double inv_h2, const double* model_partial,
                          double* partial, hdk_ctl* ctl, void* stream) {
  hdk::launch(k_tr_partials, dim3(HDK_RED_BLOCKS), dim3(kT), 0, S(stream), *x, ne, e_prev, e_star, q_prev, q_star, q_tilde, partial);
  hdk::launch(k_tr_final, dim3(1), dim3(kT), 0, S(stream), ctl, model_partial, partial, inv_h2);
  return last();
}

HDK_API int hdk_route_vertices(const hdk_vtx* x, const double* mu, const double* ef_damp, const double* b_mu,
                               const double* q_bar, const double* v_bar, const double* coup_fixed, double h,
                               double alpha, int hook_vertex, double hook_k, double hook_d, double* dl_dq_t,
                               double* dl_dv_t, double* dl_df_acc, void* stream) {
  hdk::launch(k_route_vtx, dim3(nb(x->nv)), dim3(256), 0, S(stream), *x, mu, ef_damp, b_mu, q_bar, v_bar, coup_fixed, h, alpha, hook_vertex,
                                                 hook_k, hook_d, dl_dq_t, dl_dv_t, dl_df_acc);
  return last();
}

HDK_API int hdk_fixed_coupling_t(const hdk_csr* a_df, const int* fixed, const int* p2v, const double* mu, double* coup,
                                 void* stream) {
  hdk::launch(k_fixed_coupling_t, dim3(nb(a_df->rows)), dim3(256), 0, S(stream), *a_df, fixed, p2v, mu, coup);
  return last();
}

HDK_API int hdk_axpby(int n, double a, const double* x, double b, const double* z, double* y, void* stream) {
  hdk::launch(k_axpby, dim3(nb(n)), dim3(256), 0, S(stream), n, a, x, b, z, y);
  return last();
}

HDK_API int hdk_velocity(int n, const double* q_star, const double* q_t, double h, double* v_star, void* stream) {
  hdk::launch(k_velocity, dim3(nb(n)), dim3(256), 0, S(stream), n, q_star, q_t, h, v_star);
  return last();
}

HDK_API int hdk_ctl_init(hdk_ctl* ctl, int window, double guard, int k_max, double eps_rel, double eps_abs, double tol,
                         double eps_tr, int iterations0, void* stream) {
  hdk::launch(k_ctl_init, dim3(1), dim3(1), 0, S(stream), ctl, window, guard, k_max, eps_rel, eps_abs, tol, eps_tr, iterations0);
  return last();
}

HDK_API int hdk_aa_reset(hdk_ctl* ctl, int window, double guard, int k_max, double tol, void* stream) {
  hdk::launch(k_aa_reset, dim3(1), dim3(1), 0, S(stream), ctl, window, guard, k_max, tol);
  return last();
}

HDK_API int hdk_commit(int n, const hdk_ctl* ctl, const double* q_star, double h, double* q, double* v, void* stream) {
  hdk::launch(k_commit, dim3(nb(n)), dim3(256), 0, S(stream), n, ctl, q_star, h, q, v);
  return last();
}

}  // extern "C"
