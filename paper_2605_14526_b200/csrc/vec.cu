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
#include "backbone.cuh"

HDK_TRACE_TU(vec)

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

// Block partials of the 18 Anderson quantities, stored quantity-major
// (partial[q * HDK_RED_BLOCKS + block], read by aa_solve_block), via a
// reduce-scatter butterfly (20 shuffles instead of 18 x 5; backbone.cuh).
__device__ __forceinline__ void block_partials_18(const double (&v)[18], double* partial) {
  __shared__ double sm[kT / 32][18];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int q0, len;
  const double w = hdk::warp_rs_18(v, lane, q0, len);
  if (len >= 1) sm[warp][q0] = w;
  __syncthreads();
  if (threadIdx.x < 18) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) t += sm[w][threadIdx.x];
    partial[threadIdx.x * HDK_RED_BLOCKS + blockIdx.x] = t;  // quantity-major: coalesced folds
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
      v[i] = b < HDK_RED_BLOCKS ? __ldg(partial + b * HDK_RED_Q + q) : 0.0;
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

// The same sums from forces stored by incidence slot (k_local with
// corner_vpos): contiguous reads, the same order, so bitwise gather_vtx.
__device__ __forceinline__ void gather_vtx_sorted(const hdk_vtx& x, const double* __restrict__ efs, int v, double& s0,
                                                  double& s1, double& s2) {
  s0 = s1 = s2 = 0.0;
  const int e = x.inc_off[v + 1];
#pragma unroll 4
  for (int j = x.inc_off[v]; j < e; ++j) {
    const double* p = efs + 3 * (size_t)j;
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

template <bool kSorted>
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
    if (kSorted) gather_vtx_sorted(x, ef, v, g[0], g[1], g[2]);
    else gather_vtx(x, ef, v, g[0], g[1], g[2]);
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

// k_gather_perm over the elimination-order incidence; same terms, same lane
// split and fold, so bitwise the same sums.
// sorted != 0: ef holds the forces already in incidence order (hdk_bapply_sorted),
// so the range is read directly.
__device__ __forceinline__ void gather_pp_body(hdk_vtx x, const double* __restrict__ basep, const double* __restrict__ ef,
                            double* __restrict__ rhs, const int* run_flag, int sorted) {
  HDK_TRACED_WAIT(hdk::kTrGather);
  hdk::pdl_trigger();
  if (run_flag && *run_flag == 0) return;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = gid >> 3, sub = gid & 7;
  const bool live = p < x.n;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  if (live) {
    const int e = __ldg(x.pinc_off + p + 1);
#pragma unroll 4
    for (int j = __ldg(x.pinc_off + p) + sub; j < e; j += 8) {
      const double* q = ef + 3 * (size_t)(sorted ? j : __ldg(x.pinc + j));
      s0 += __ldg(q);
      s1 += __ldg(q + 1);
      s2 += __ldg(q + 2);
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (live && sub == 0) {
    rhs[3 * (size_t)p] = (basep ? basep[3 * (size_t)p] : 0.0) + s0;
    rhs[3 * (size_t)p + 1] = (basep ? basep[3 * (size_t)p + 1] : 0.0) + s1;
    rhs[3 * (size_t)p + 2] = (basep ? basep[3 * (size_t)p + 2] : 0.0) + s2;
  }
}
__global__ void k_gather_pp(hdk_vtx x, const double* __restrict__ basep, const double* __restrict__ ef,
                            double* __restrict__ rhs, const int* run_flag, int sorted) {
  gather_pp_body(x, basep, ef, rhs, run_flag, sorted);
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
  block_partials_18(acc, partial);
}

// Anderson coefficient solve (forward.cpp:31-47): M gamma = DG^T g with
// M = DG^T DG + 1e-6 |DG|_F^2 / window I, by LDL^T with Eigen::LDLT's
// diagonal pivoting (left-looking; pivots chosen on the untouched diagonal).
// Runs on one block of kT threads (inside k_aa_solve, or as the tail of
// k_aa_dots_fused in the block that finishes last): all warps fold the
// partial sums with every load in flight at once, then warp 0 alone does the
// bookkeeping and the factorization in registers — lane i holds row i of the
// Gram matrix and row rank(i) of L, pivot rows travel by shuffle, and the
// pivot order, d and the substitution values are warp-uniform.  mode 1 also
// evaluates the adjoint convergence test first (backward.cpp:191-193) and
// sets the WHILE condition (graph handle given).
constexpr int kSolveT = kT;
constexpr int kNQ = 2 * HDK_AA_MAX + 2;
// Barrier of threads 0..63 only (the factorization warps).
__device__ __forceinline__ void named_bar64() { asm volatile("bar.sync 2, 64;" ::: "memory"); }

// What the mixing step of the calling block needs from the solve (shared).
struct AaResult {
  double gamma[HDK_AA_MAX];
  double gslot[HDK_AA_MAX];  // gamma by history ring slot (0 for unused slots)
  int done, mixed, count, head, window, err;
};

// State is read from `in` and the updated state written to `out` (NULL: not
// written), so a kernel whose every block solves redundantly can read a
// snapshot while one block publishes (k_bb_mix).  `res` (shared memory,
// optional) receives the mixing inputs for the calling block.
__device__ __noinline__ void aa_solve_block(const hdk_ctl* in, hdk_ctl* gctl, const double* partial, int mode,
                                            cudaGraphConditionalHandle handle, int use_handle,
                                            AaResult* res = nullptr) {
  constexpr int M = HDK_AA_MAX;
  __shared__ double s[kNQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp 0: control scalars and its Gram rows, loaded ahead of the fold
  int m = 1, count = 0, head = 0, has_last = 0, mixed = 0, kk = 0, iters = 0, err = 0, done = 0, k_max = 0;
  double tol = 0.0, guard = 0.0;
  double g[M];
  if (warp == 0) {
    m = in->window; count = in->count; head = in->head; has_last = in->has_last; mixed = in->mixed;
    kk = in->k; iters = in->iterations; err = in->err; done = in->done; k_max = in->k_max;
    tol = in->tol; guard = in->guard;
#pragma unroll
    for (int j = 0; j < M; ++j) g[j] = lane < M ? in->gram[lane * M + j] : 0.0;
  }
  {  // fold: warp w owns quantities w, w + 8, w + 16; all loads issued first
    constexpr int R = (kNQ + kT / 32 - 1) / (kT / 32);
    double v[R][kFoldPerLane];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = warp + r * (kT / 32);
#pragma unroll
      for (int i = 0; i < kFoldPerLane; ++i) {
        const int b = lane + 32 * i;
        v[r][i] = (q < kNQ && b < HDK_RED_BLOCKS) ? partial[q * HDK_RED_BLOCKS + b] : 0.0;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double t = 0.0;
#pragma unroll
      for (int i = 0; i < kFoldPerLane; ++i) t += v[r][i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      const int q = warp + r * (kT / 32);
      if (lane == 0 && q < kNQ) s[q] = t;
    }
  }
  __syncthreads();
  hdk::trace_stamp(g_hdk_trace, hdk::kTrTail1);
  // ---- warp 0: convergence test, history bookkeeping, pivot order ----------
  __shared__ double sG[M][M + 1], sA[M][M + 1], sd[M], sy[M], sgam[M];
  __shared__ int sperm[M], sn, sok;
  __shared__ double sridge;
  const unsigned F = 0xffffffffu;
  bool skip = false;
  int nsol = 0;
  double gam[M];
#pragma unroll
  for (int c = 0; c < M; ++c) gam[c] = 0.0;
  if (warp == 0) {
    if (mode == 1) {  // adjoint backbone: convergence test before mixing
      iters += 1;
      const double diff = sqrt(s[2 * M]);
      const double base = fmax(sqrt(s[2 * M + 1]), 1e-30);
      kk += 1;
      if (diff <= tol * base) {
        done = 1;
        mixed = 0;
        skip = true;
      } else if (kk >= k_max && err == 0) {
        err = 10;  // AdjointDiverged (cap)
      }
    }
    int n = 0;
    if (!skip) {
      if (has_last) {
        if (count < m) {
          count += 1;
        } else {  // drop the oldest: gram[i][j] <- gram[i+1][j+1]
          head = (head + 1) % m;
          double nx[M];
#pragma unroll
          for (int j = 0; j < M; ++j) nx[j] = __shfl_down_sync(F, g[j], 1);
#pragma unroll
          for (int j = 0; j + 1 < M; ++j) g[j] = nx[j + 1];
        }
        const int j0 = count - 1;  // newest row / column = DG^T dg_new
#pragma unroll
        for (int j = 0; j < M; ++j)
          if (j == j0 && lane < count) g[j] = s[lane];
        if (lane == j0)
#pragma unroll
          for (int l = 0; l < M; ++l)
            if (l < count) g[l] = s[l];
      }
      has_last = 1;
      mixed = 0;
      n = count;
    }
    double mydiag = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j)
      if (j == lane) mydiag = g[j];
    double fro2 = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const double dj = __shfl_sync(F, mydiag, j);
      if (j < n) fro2 += dj;
    }
    if (n > 0 && fro2 > 0.0) {
      nsol = n;
      const double ridge = 1e-6 * fro2 / m;
      // pivot order: largest |diagonal| among the remaining untouched ones,
      // swapped into place (Eigen LDLT).  With distinct |diagonals| that is
      // the descending order, found by ranks in one pass; ties (which the
      // swaps resolve position-dependently) take the serial selection.
      const double ad = lane < n ? fabs(mydiag + ridge) : -1.0;
      int rank = 0;
      bool tie = false;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const double aj = __shfl_sync(F, ad, j);
        if (j < n && lane < n) {
          if (aj > ad) ++rank;
          else if (aj == ad && j != lane) tie = true;
        }
      }
      if (!__any_sync(F, tie)) {
        if (lane < n) sperm[rank] = lane;
      } else {
        int perm[M];
        double dv[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
          perm[i] = i;
          dv[i] = __shfl_sync(F, mydiag, i) + ridge;
        }
#pragma unroll
        for (int k = 0; k < M; ++k) {
          if (k < n) {
            int piv = k;
            double best = fabs(dv[k]);
#pragma unroll
            for (int i = k + 1; i < M; ++i)
              if (i < n && fabs(dv[i]) > best) {
                best = fabs(dv[i]);
                piv = i;
              }
            const int pk = perm[k];
            const double dk = dv[k];
            int pp = pk;
            double dp = dk;
#pragma unroll
            for (int i = k + 1; i < M; ++i)
              if (i == piv) {
                pp = perm[i];
                dp = dv[i];
                perm[i] = pk;
                dv[i] = dk;
              }
            perm[k] = pp;
            dv[k] = dp;
          }
        }
#pragma unroll
        for (int i = 0; i < M; ++i)
          if (lane == i) sperm[i] = perm[i];
      }
      if (lane == 0) sridge = ridge;
      if (lane < M)
#pragma unroll
        for (int j = 0; j < M; ++j) sG[lane][j] = g[j];
    }
    if (lane == 0) sn = nsol;
  }
  hdk::trace_stamp(g_hdk_trace, hdk::kTrTail3);
  __syncthreads();
  // ---- threads 0..63: LDL^T of the permuted matrix in shared memory ---------
  // Right-looking with the left-looking (Eigen) operation order per entry:
  // A(i,k) -= (L(i,l) L(k,l)) d(l) for l = 0, 1, ...; then L(i,k) = A(i,k) / d(k).
  const int ns = sn;
  if (ns > 0 && threadIdx.x < 64) {
    const int i = threadIdx.x >> 3, j = threadIdx.x & 7;
    if (i < ns && j < ns) sA[i][j] = sG[sperm[i]][sperm[j]] + (i == j ? sridge : 0.0);
    if (threadIdx.x == 0) sok = 1;
    named_bar64();
    for (int k = 0; k < ns; ++k) {
      const double dk = sA[k][k];
      if (j == k && i > k && i < ns) sA[i][k] = sA[i][k] / dk;  // L(i,k)
      if (threadIdx.x == 0) {
        sd[k] = dk;
        if (!(fabs(dk) > 2.2250738585072014e-308)) sok = 0;
      }
      named_bar64();
      if (i > k && i < ns && j > k && j <= i) sA[i][j] -= sA[i][k] * sA[j][k] * dk;
      named_bar64();
    }
    // y = L^{-1} P b (row order of subtractions as in the serial form)
    const int t = threadIdx.x;
    if (t < ns) sy[t] = s[M + sperm[t]];
    named_bar64();
    for (int k = 0; k < ns; ++k) {
      if (t > k && t < ns) sy[t] -= sA[t][k] * sy[k];
      named_bar64();
    }
    if (t < ns) sy[t] /= sd[t];
    named_bar64();
    for (int k = ns - 1; k > 0; --k) {  // L^T x = y, column-oriented
      if (t < k) sy[t] -= sA[k][t] * sy[k];
      named_bar64();
    }
    if (t < ns) sgam[sperm[t]] = sy[t];
  }
  hdk::trace_stamp(g_hdk_trace, hdk::kTrTail4);
  __syncthreads();
  if (warp != 0) return;
  if (nsol > 0) {
#pragma unroll
    for (int c = 0; c < M; ++c) gam[c] = c < nsol ? sgam[c] : 0.0;
    bool good = sok != 0;
#pragma unroll
    for (int i = 0; i < M; ++i)
      if (i < nsol) good = good && isfinite(gam[i]);
    double gn = 0.0;
    if (good)
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (i < nsol) gn += gam[i] * gam[i];
    if (!good || !(sqrt(gn) <= guard)) {  // guard: discard history (forward.cpp:43-47)
      count = 0;
      head = 0;
      has_last = 0;
      nsol = 0;
    } else {
      mixed = 1;
    }
  }
  hdk::trace_stamp(g_hdk_trace, hdk::kTrTail2);
  if (res && lane == 0) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
      res->gamma[i] = gam[i];
      res->gslot[i] = 0.0;
    }
    if (mixed)
      for (int j = 0; j < count; ++j) res->gslot[(head + j) % m] = gam[j];
    res->done = done;
    res->mixed = mixed;
    res->count = count;
    res->head = head;
    res->window = m;
    res->err = err;
  }
  if (!gctl) return;
  if (lane < M)
#pragma unroll
    for (int j = 0; j < M; ++j) gctl->gram[lane * M + j] = g[j];
  if (lane == 0) {
    if (nsol > 0)
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (i < nsol) gctl->gamma[i] = gam[i];
    gctl->count = count;
    gctl->head = head;
    gctl->has_last = has_last;
    gctl->mixed = mixed;
    gctl->k = kk;
    gctl->iterations = iters;
    gctl->err = err;
    gctl->done = done;
    if (mode == 1) {  // adjoint loop condition (done / error)
      const int cond = (!done && err == 0) ? 1 : 0;
      gctl->cond = cond;
      if (use_handle) cudaGraphSetConditional(handle, cond);
    }
  }
}

__global__ void __launch_bounds__(kSolveT) k_aa_solve(hdk_ctl* gctl, const double* partial, int mode) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  aa_solve_block(gctl, gctl, partial, mode, 0, 0);
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
    const int2 vf = __ldg(f.vfold + v);
    double th;
    if (vf.y > 0) {  // slots of consecutive CTAs are one tile (256 columns) apart
      th = 0.0;
      for (int b = 0; b < vf.y; ++b) th += __ldg(f.part2 + 3 * ((size_t)vf.x + 256 * (size_t)b) + a);
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
  static_assert(2 * HDK_AA_MAX + 2 == 18, "butterfly sized for window 8");
  block_partials_18(acc, partial);
  // last block folds every partial and runs the coefficient solve; only the
  // partial writers need their stores visible before the ticket
  if (mode & 256) return;  // profiling ablation: no tail
  __shared__ int is_last;
  if (threadIdx.x < 18) __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(ticket, 1u);
    is_last = t == gridDim.x - 1;
    if (is_last) *ticket = 0u;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  aa_solve_block(ctl, ctl, partial, mode, handle, use_handle);
}

__global__ void k_trace_epoch(unsigned long long* buf) {  // advance and clear the next record slot
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const unsigned long long ep = buf[0] + 1ULL;
  unsigned long long* r = buf + 1 + 3 * ((ep % hdk::kTraceSlots) * hdk::kTrCount);
  for (int i = 0; i < hdk::kTrCount; ++i) {
    r[3 * i] = ~0ULL;
    r[3 * i + 1] = ~0ULL;
    r[3 * i + 2] = 0ULL;
  }
  __threadfence();
  buf[0] = ep;
}

// True in the block that arrives last.  The CTA barrier orders every
// thread's partial stores before thread 0's acq_rel ticket (release), and the
// last block's acquire orders its later loads of the others' partials — one
// L2 round trip instead of an SC fence plus an atomic.
__device__ __forceinline__ bool last_block_ticket(unsigned int* ticket) {
  __shared__ int is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(ticket) : "memory");
    is_last = t == gridDim.x - 1;
    if (is_last) asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(ticket) : "memory");
  }
  __syncthreads();
  return is_last != 0;
}

// Refill loop of the contact-adjoint columns: continue while every column
// that was iterating at launch still is (*expected of them), so the loop
// exits right after a column finishes and the host hands its slot the next
// contact row.  *any doubles as the solve's run flag.
__global__ void k_cols_cond(const hdk_ctl* ctls, int count, const int* expected, int* any,
                            cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int c = threadIdx.x;
  const int on = c < count && ctls[c].cond != 0 && ctls[c].err == 0 && ctls[c].nonfinite == 0;
  const int active = __popc(__ballot_sync(0xffffffffu, on));
  if (threadIdx.x == 0) {
    const int a = (active > 0 && active == *expected) ? 1 : 0;
    *any = a;
    if (use_handle) cudaGraphSetConditional(handle, a);
  }
}

// OR of several backbone loops' conditions (multi-column contact adjoint).
__global__ void k_any_cond(const hdk_ctl* ctls, int count, int* any, cudaGraphConditionalHandle handle,
                           int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int c = threadIdx.x;
  const int on = c < count && ctls[c].cond != 0 && ctls[c].err == 0 && ctls[c].nonfinite == 0;
  const int a = __any_sync(0xffffffffu, on) ? 1 : 0;
  if (threadIdx.x == 0) {
    *any = a;
    if (use_handle) cudaGraphSetConditional(handle, a);
  }
}

// ---- adjoint backbone in elimination order -----------------------------------
// The backbone's Anderson vectors (t, x, last, history) live in elimination
// order [n][3]: the solve's tile partials fold into t with contiguous loads,
// and every Anderson access is coalesced with no vertex indirection.  Fixed
// vertices carry t = x = 0 in the backbone (they contribute nothing to any
// dot product), so dropping them changes no value, only the summation order.
// i0 / nseg3: the index range of one sample of a segmented batch (the
// history rings keep the whole vector's stride n3); a single problem passes
// 0 / 3 n.
__device__ __forceinline__ void bb_dots_body(int n, hdk_factor f, hdk_ctl* ctl, hdk_ctl* snap, double* __restrict__ tp,
                                                double* __restrict__ tv, const double* __restrict__ xp, double* last_q,
                                                double* last_g, double* dq, double* dg, double* partial, int mode,
                                                size_t i0 = 0, size_t nseg3 = 0) {
  HDK_TRACED_WAIT(hdk::kTrDots);
  hdk::pdl_trigger();
  const size_t n3 = 3 * (size_t)n;
  if (blockIdx.x == 0) {  // snapshot of the control block for k_bb_mix (which rewrites ctl)
    if (threadIdx.x == 0 && ctl->nonfinite && ctl->err == 0) {  // AdjointDiverged
      ctl->err = 10;
      ctl->cond = 0;
    }
    __syncthreads();
    const int* src = reinterpret_cast<const int*>(ctl);
    int* dst = reinterpret_cast<int*>(snap);
    for (int w = threadIdx.x; w < static_cast<int>(sizeof(hdk_ctl) / 4); w += kT) dst[w] = src[w];
  }
  if (ctl->cond == 0) return;  // unrolled iteration past convergence (the snapshot still carries cond = 0)
  hdk::BbState st = hdk::bb_state(ctl);
  if (mode & 512) st.c2 = 0;  // profiling ablation
  const hdk::BbArgs args{ctl, tp, tv, xp, last_q, last_g, dq, dg};
  double acc[2 * HDK_AA_MAX + 2];
#pragma unroll
  for (int q = 0; q < 2 * HDK_AA_MAX + 2; ++q) acc[q] = 0.0;
  const unsigned long long pol = hdk::pol_keep();
  const size_t iend = i0 + (nseg3 ? nseg3 : n3);
  for (size_t i = i0 + blockIdx.x * kT + threadIdx.x; i < iend; i += (size_t)gridDim.x * kT) {
    const int col = static_cast<int>(i / 3), a = static_cast<int>(i - 3 * (size_t)col);
    const hdk::BbIn pre = hdk::bb_prefetch(args, st, n3, i, pol);
    const int tile = col >> 8;  // tile_cta2 is tiny and L1-resident
    const int tb0 = __ldg(f.tile_cta2 + 2 * tile), tb1 = __ldg(f.tile_cta2 + 2 * tile + 1);
    int2 pf = make_int2((tile + tb0) * 256 + (col & 255), tb1 - tb0 + 1);
    double th = 0.0;
    if (mode & 1024) pf.y = 0;  // profiling ablation
    for (int b0 = 0; b0 < pf.y; b0 += 4) {  // loads first, then the fixed-order adds
      double v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        v[k] = b0 + k < pf.y ? __ldg(f.part2 + 3 * ((size_t)pf.x + 256 * (size_t)(b0 + k)) + a) : 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (b0 + k < pf.y) th += v[k];
    }
    hdk::bb_dots_elem(args, st, pre, f.p2v, n3, i, th, acc, pol);
  }
  static_assert(2 * HDK_AA_MAX + 2 == 18, "butterfly sized for window 8");
  hdk::trace_stamp(g_hdk_trace, hdk::kTrDotsA);
  block_partials_18(acc, partial);
  hdk::trace_stamp(g_hdk_trace, hdk::kTrDotsB);
}
__global__ void __launch_bounds__(kT) k_bb_dots(int n, hdk_factor f, hdk_ctl* ctl, hdk_ctl* snap, double* __restrict__ tp,
                                                double* __restrict__ tv, const double* __restrict__ xp, double* last_q,
                                                double* last_g, double* dq, double* dg, double* partial, int mode) {
  bb_dots_body(n, f, ctl, snap, tp, tv, xp, last_q, last_g, dq, dg, partial, mode);
}

// x <- t - sum_j gamma_j (dq_j + dg_j) in elimination order, also scattered to
// the full vertex vector the element kernels read.
// Anderson coefficient solve of the backbone on its own graph branch (one
// block): runs while B t and its gather proceed on the main branch, reads
// the snapshot k_bb_dots took, publishes the new state and the WHILE
// condition to ctl and the mixing inputs to *res.
__device__ __forceinline__ void bb_solve_body(hdk_ctl* ctl, const hdk_ctl* snap, const double* partial,
                                                 AaResult* out, cudaGraphConditionalHandle handle, int use_handle) {
  HDK_TRACED_WAIT(hdk::kTrTail0);
  hdk::pdl_trigger();
  if (snap->cond == 0) return;  // unrolled iteration past convergence
  __shared__ AaResult res;
  aa_solve_block(snap, ctl, partial, 1, handle, use_handle, &res);
  __syncthreads();
  const int* src = reinterpret_cast<const int*>(&res);
  int* dst = reinterpret_cast<int*>(out);
  for (int w = threadIdx.x; w < static_cast<int>(sizeof(AaResult) / 4); w += kT) dst[w] = src[w];
}
__global__ void __launch_bounds__(kT) k_bb_solve(hdk_ctl* ctl, const hdk_ctl* snap, const double* partial,
                                                 AaResult* out, cudaGraphConditionalHandle handle, int use_handle) {
  bb_solve_body(ctl, snap, partial, out, handle, use_handle);
}

// Anderson mix of the backbone, in elimination order, carried in two spaces:
//   x_{k+1} = t_k - sum_j gamma_j (dq_j + dg_j)                 (backward.cpp:188-199)
//   R(x_{k+1}) = R(t_k) - sum_j gamma_j R(dq_j + dg_j),  R = gather o B,
// by linearity of R, so the next right-hand side seed + R(x_{k+1}) is ready
// without applying B to the mixed iterate (B t_k ran beside the coefficient
// solve).  The rings hold the sums s_j = dq_j + dg_j (k_bb_dots) and their
// R-images (pushed here from the tracked R(x_k) and R(t_k), same slots); a
// history reset restarts the R side from R(t_k) exactly.
__device__ __forceinline__ void bb_mix_body(int n, const int* __restrict__ p2v, hdk_ctl* ctl, const hdk_ctl* snap,
                                               const AaResult* __restrict__ res, const double* __restrict__ tp,
                                               double* xp, double* __restrict__ xv, const double* __restrict__ sq,
                                               const double* __restrict__ rt, double* rx, double* last_rx,
                                               double* last_rg, double* rsq, const double* __restrict__ seedp,
                                               double* __restrict__ rhs, size_t i0 = 0, size_t nseg3 = 0) {
  HDK_TRACED_WAIT(hdk::kTrMix);
  hdk::pdl_trigger();
  if (snap->cond == 0) return;  // unrolled iteration past convergence
  const size_t n3 = 3 * (size_t)n;
  const size_t il = blockIdx.x * (size_t)kT + threadIdx.x;
  if (il >= (nseg3 ? nseg3 : n3)) return;
  const size_t i = i0 + il;
  const unsigned long long pol = hdk::pol_keep();
  // ring slot of the entry pushed this iteration (state before the update, as k_bb_dots)
  const int m = snap->window, c0 = snap->count, h0 = snap->head;
  const bool push = snap->has_last != 0;
  const int ns = push ? (c0 < m ? (h0 + c0) % m : h0) : -1;
  const bool done = res->done != 0;
  const int mixed = res->mixed, c = res->count;
  double hs[HDK_AA_MAX], rs[HDK_AA_MAX];
#pragma unroll
  for (int sl = 0; sl < HDK_AA_MAX; ++sl) {
    hs[sl] = sl < m ? hdk::ld_keep(sq + sl * n3 + i, pol) : 0.0;
    rs[sl] = sl < m && sl != ns ? hdk::ld_keep(rsq + sl * n3 + i, pol) : 0.0;
  }
  const double qc = hdk::ld_keep(xp + i, pol), th = hdk::ld_keep(tp + i, pol);
  const double rxc = hdk::ld_keep(rx + i, pol), rth = hdk::ld_keep(rt + i, pol);
  const double rgn = rth - rxc;
  if (push) {
    const double rdqn = rxc - hdk::ld_keep(last_rx + i, pol);
    const double rdgn = rgn - hdk::ld_keep(last_rg + i, pol);
    const double rsn = rdqn + rdgn;
    hdk::st_keep(rsq + ns * n3 + i, rsn, pol);
#pragma unroll
    for (int sl = 0; sl < HDK_AA_MAX; ++sl)
      if (sl == ns) rs[sl] = rsn;
  }
  hdk::st_keep(last_rx + i, rxc, pol);
  hdk::st_keep(last_rg + i, rgn, pol);
  double out = qc + (th - qc), rout = rxc + rgn;
  if (done) {
    out = th;
    rout = rth;
  } else if (mixed) {  // valid ring slots are 0..count-1 (head moves only once the ring is full)
#pragma unroll
    for (int sl = 0; sl < HDK_AA_MAX; ++sl)
      if (sl < c) {
        out -= res->gslot[sl] * hs[sl];
        rout -= res->gslot[sl] * rs[sl];
      }
  }
  hdk::st_keep(xp + i, out, pol);
  hdk::st_keep(rx + i, rout, pol);
  rhs[i] = seedp[i] + rout;
  const int col = static_cast<int>(i / 3);
  xv[3 * (size_t)__ldg(p2v + col) + (i - 3 * (size_t)col)] = out;
  if (!isfinite(out) || !isfinite(rout)) atomicOr(&ctl->nonfinite, 1);
}
__global__ void __launch_bounds__(kT) k_bb_mix(int n, const int* __restrict__ p2v, hdk_ctl* ctl, const hdk_ctl* snap,
                                               const AaResult* __restrict__ res, const double* __restrict__ tp,
                                               double* xp, double* __restrict__ xv, const double* __restrict__ sq,
                                               const double* __restrict__ rt, double* rx, double* last_rx,
                                               double* last_rg, double* rsq, const double* __restrict__ seedp,
                                               double* __restrict__ rhs) {
  bb_mix_body(n, p2v, ctl, snap, res, tp, xp, xv, sq, rt, rx, last_rx, last_rg, rsq, seedp, rhs);
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
  c->window = window < 1 ? 1 : window; c->count = 0; c->head = 0; c->has_last = 0; c->mixed = 0; c->nonfinite = 0;
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
  c->window = window < 1 ? 1 : window; c->count = 0; c->head = 0; c->has_last = 0; c->mixed = 0; c->nonfinite = 0;
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


// ---- contact-adjoint columns, one launch per stage for all columns ---------
// blockIdx.y selects the column (hdk_bb_columns); the bodies are the
// single-column kernels', so every column computes exactly what its own
// launch would.
__global__ void __launch_bounds__(kT) k_bb_dots_cols(int n, hdk_bb_columns c, int mode) {
  const hdk_bb_column& k = c.col[blockIdx.y];
  bb_dots_body(n, k.f, k.ctl, k.snap, k.t, k.tv, k.xp, k.lastq, k.lastg, k.dq, k.dg, k.part, mode);
}
__global__ void __launch_bounds__(kT) k_bb_solve_cols(hdk_bb_columns c) {
  const hdk_bb_column& k = c.col[blockIdx.x];
  bb_solve_body(k.ctl, k.snap, k.part, static_cast<AaResult*>(k.res), 0ULL, 0);
}
__global__ void k_gather_pp_cols(hdk_vtx x, hdk_bb_columns c) {
  const hdk_bb_column& k = c.col[blockIdx.y];
  gather_pp_body(x, nullptr, k.ef, k.rt, &k.snap->cond, 0);
}
__global__ void __launch_bounds__(kT) k_bb_mix_cols(int n, const int* __restrict__ p2v, hdk_bb_columns c) {
  const hdk_bb_column& k = c.col[blockIdx.y];
  bb_mix_body(n, p2v, k.ctl, k.snap, static_cast<const AaResult*>(k.res), k.t, k.xp, k.x, k.dq, k.rt, k.rx, k.lrx,
              k.lrg, k.rsq, k.seedp, k.rhs);
}

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
  hdk::launch(k_gather_rhs<false>, dim3(HDK_RED_BLOCKS), dim3(kT), 0, S(stream), *x, ef, inv_h2, q_tilde, damp, fixcoup, b_prev, rhs_perm, partial);
  return last();
}
HDK_API int hdk_gather_rhs_sorted(const hdk_vtx* x, const double* efs, double inv_h2, const double* q_tilde,
                                  const double* damp, const double* fixcoup, double* b_prev, double* rhs_perm,
                                  double* partial, void* stream) {
  hdk::launch(k_gather_rhs<true>, dim3(HDK_RED_BLOCKS), dim3(kT), 0, S(stream), *x, efs, inv_h2, q_tilde, damp, fixcoup, b_prev, rhs_perm, partial);
  return last();
}

HDK_API int hdk_gather_perm(const hdk_vtx* x, const double* base, const double* ef, double* rhs_perm, void* stream) {
  hdk::launch(k_gather_perm, dim3(nb(8LL * x->n)), dim3(256), 0, S(stream), *x, base, ef, rhs_perm);
  return last();
}

HDK_API int hdk_gather_pp(const hdk_vtx* x, const double* base_perm, const double* ef, double* rhs_perm,
                          const int* run_flag, void* stream) {
  if (!x->pinc_off || !x->pinc) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_gather_pp, dim3(nb(8LL * x->n)), dim3(256), 0, S(stream), *x, base_perm, ef, rhs_perm, run_flag, 0);
  return last();
}

HDK_API int hdk_gather_sorted(const hdk_vtx* x, const double* base_perm, const double* ef_sorted, double* rhs_perm,
                              const int* run_flag, void* stream) {
  if (!x->pinc_off) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_gather_pp, dim3(nb(8LL * x->n)), dim3(256), 0, S(stream), *x, base_perm, ef_sorted, rhs_perm, run_flag, 1);
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
  if (!f->vfold || g2 != f->grid2) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_aa_dots_fused, dim3(HDK_RED_BLOCKS), dim3(kT), 0, S(stream), *x, *f, g2, ctl, qhat, qcur, last_q,
              last_g, dq, dg, partial, ticket, mode, static_cast<cudaGraphConditionalHandle>(cond_handle),
              cond_handle != 0ULL ? 1 : 0);
  return last();
}

HDK_API int hdk_trace_epoch(unsigned long long* buf, void* stream) {
  hdk::launch(k_trace_epoch, dim3(1), dim3(1), 0, S(stream), buf);
  return last();
}

HDK_API int hdk_cols_cond(hdk_ctl* ctls, int count, const int* expected, int* any, unsigned long long cond_handle,
                          void* stream) {
  hdk::launch(k_cols_cond, dim3(1), dim3(32), 0, S(stream), ctls, count, expected, any,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle != 0ULL ? 1 : 0);
  return last();
}

HDK_API int hdk_any_cond(hdk_ctl* ctls, int count, int* any, unsigned long long cond_handle, void* stream) {
  hdk::launch(k_any_cond, dim3(1), dim3(32), 0, S(stream), ctls, count, any,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle != 0ULL ? 1 : 0);
  return last();
}

HDK_API int hdk_bb_dots(const hdk_factor* f, hdk_ctl* ctl, hdk_ctl* snap, double* t_perm, double* t_full,
                        const double* x_perm, double* last_q, double* last_g, double* dq, double* dg, double* partial,
                        int mode, void* stream) {
  int g1 = 0, g2 = 0;
  hdk_solve_grids(f, &g1, &g2);
  if (!f->tile_cta2 || g2 != f->grid2) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_bb_dots, dim3(HDK_RED_BLOCKS), dim3(kT), 0, S(stream), f->n, *f, ctl, snap, t_perm, t_full, x_perm,
              last_q, last_g, dq, dg, partial, mode);
  return last();
}

HDK_API int hdk_bb_solve(hdk_ctl* ctl, const hdk_ctl* snap, const double* partial, void* result,
                         unsigned long long cond_handle, void* stream) {
  hdk::launch(k_bb_solve, dim3(1), dim3(kT), 0, S(stream), ctl, snap, partial, static_cast<AaResult*>(result),
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle != 0ULL ? 1 : 0);
  return last();
}

HDK_API size_t hdk_bb_result_bytes(void) { return sizeof(AaResult); }

HDK_API int hdk_bb_mix(const hdk_factor* f, hdk_ctl* ctl, const hdk_ctl* snap, const void* result,
                       const double* t_perm, double* x_perm, double* x_full, const double* sum_hist,
                       const double* rt_perm, double* rx_perm, double* last_rx, double* last_rg, double* rsum_hist,
                       const double* seed_perm, double* rhs_perm, void* stream) {
  hdk::launch(k_bb_mix, dim3(nb(3LL * f->n)), dim3(kT), 0, S(stream), f->n, f->p2v, ctl, snap,
              static_cast<const AaResult*>(result), t_perm, x_perm, x_full, sum_hist, rt_perm, rx_perm, last_rx,
              last_rg, rsum_hist, seed_perm, rhs_perm);
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


HDK_API int hdk_bb_columns_dots(const hdk_bb_columns* c, int mode, void* stream) {
  const hdk_factor* f = &c->col[0].f;
  int g1 = 0, g2 = 0;
  hdk_solve_grids(f, &g1, &g2);
  if (!f->tile_cta2 || g2 != f->grid2) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_bb_dots_cols, dim3(HDK_RED_BLOCKS, HDK_BB_COLUMNS), dim3(kT), 0, S(stream), f->n, *c, mode);
  return last();
}
HDK_API int hdk_bb_columns_solve(const hdk_bb_columns* c, void* stream) {
  hdk::launch(k_bb_solve_cols, dim3(HDK_BB_COLUMNS), dim3(kT), 0, S(stream), *c);
  return last();
}
HDK_API int hdk_bb_columns_gather(const hdk_vtx* x, const hdk_bb_columns* c, void* stream) {
  if (!x->pinc_off || !x->pinc) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_gather_pp_cols, dim3(nb(8LL * x->n), HDK_BB_COLUMNS), dim3(256), 0, S(stream), *x, *c);
  return last();
}
HDK_API int hdk_bb_columns_mix(const hdk_bb_columns* c, void* stream) {
  const hdk_factor* f = &c->col[0].f;
  hdk::launch(k_bb_mix_cols, dim3(nb(3LL * f->n), HDK_BB_COLUMNS), dim3(kT), 0, S(stream), f->n, f->p2v, *c);
  return last();
}
}  // extern "C"

// ---- segmented batch: per-sample reductions and loop control ---------------
// (hdk.h "segmented batch"; the lockstep C5 engine, engine.cpp segments > 1).
// Sample s = blockIdx.y; its blocks stride over its own index range, so each
// sample's sums are fixed-order and independent of the others.
namespace {

constexpr int kRB = HDK_SEG_RB;
constexpr size_t kPS = HDK_SEG_PSTRIDE;

// Fold of block-major partials (partial[b * HDK_RED_Q + q]) over kRB blocks.
__device__ __forceinline__ void fold_rb(const double* __restrict__ partial, int nq, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int q = warp; q < nq; q += nw) {
    double v = lane < kRB ? partial[lane * HDK_RED_Q + q] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) out[q] = v;
  }
}

__device__ __forceinline__ void ctl_init_one(hdk_ctl* c, int window, double guard, int k_max, double er, double ea,
                                             double tol, double eps_tr) {
  c->k = 0; c->k_max = k_max; c->iterations = 0; c->converged = 0;
  c->err = 0; c->done = 0; c->bad = 0; c->cond = 1;
  c->window = window < 1 ? 1 : window; c->count = 0; c->head = 0; c->has_last = 0; c->mixed = 0; c->nonfinite = 0;
  c->eps_rel = er; c->eps_abs = ea; c->guard = guard; c->tol = tol;
  c->tau = 1.0; c->rho = 1.0; c->model = 0.0; c->eps_tr = eps_tr;
  for (int i = 0; i < HDK_AA_MAX; ++i) c->gamma[i] = 0.0;
  for (int i = 0; i < HDK_AA_MAX * HDK_AA_MAX; ++i) c->gram[i] = 0.0;
}

__global__ void k_seg_ctl_init(hdk_ctl* ctl, hdk_segs g, const int* windows, double guard, int k_max, double er,
                               double ea, double tol, double eps_tr, int* any) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  for (int s = threadIdx.x; s < g.count; s += blockDim.x)
    ctl_init_one(ctl + s, windows[s], guard, k_max, er, ea, tol, eps_tr);
  if (threadIdx.x == 0) *any = 1;
}

__global__ void k_seg_aa_reset(hdk_ctl* ctl, hdk_segs g, int window, double guard, int k_max, double tol, int* any) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  for (int s = threadIdx.x; s < g.count; s += blockDim.x) {
    hdk_ctl* c = ctl + s;
    c->k = 0; c->k_max = k_max; c->iterations = 0; c->converged = 0; c->done = 0; c->cond = 1;
    c->window = window < 1 ? 1 : window; c->count = 0; c->head = 0; c->has_last = 0; c->mixed = 0; c->nonfinite = 0;
    c->guard = guard; c->tol = tol;
  }
  if (threadIdx.x == 0) *any = 1;
}

template <bool kSorted>
__global__ void __launch_bounds__(kT) k_seg_gather_rhs(hdk_vtx x, hdk_segs g, const double* __restrict__ ef,
                                                       double inv_h2, const double* __restrict__ qt,
                                                       const double* __restrict__ damp, double* bprev, double* rhs,
                                                       double* partial, const hdk_ctl* ctl) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int s = blockIdx.y;
  if (ctl[s].cond == 0) return;
  double acc[2] = {0.0, 0.0};
  const int v0 = s * g.nv, v1 = v0 + g.nv;
  for (int v = v0 + blockIdx.x * kT + threadIdx.x; v < v1; v += gridDim.x * kT) {
    const int p = x.v2p[v];
    const double m = x.mass[v];
    double gg[3];
    if (kSorted) gather_vtx_sorted(x, ef, v, gg[0], gg[1], gg[2]);
    else gather_vtx(x, ef, v, gg[0], gg[1], gg[2]);
    for (int a = 0; a < 3; ++a) {
      const size_t i = 3 * (size_t)v + a;
      double b = m * qt[i] * inv_h2;
      b += gg[a];
      b += damp[i];
      const double d = b - bprev[i];
      acc[0] += d * d;
      acc[1] += b * b;
      bprev[i] = b;
      if (p >= 0) rhs[3 * (size_t)p + a] = b;
    }
  }
  block_partials<2>(acc, partial + s * kPS);
}

__global__ void __launch_bounds__(kT) k_seg_aa_dots_fused(hdk_vtx x, hdk_factor f, hdk_segs g, hdk_ctl* ctls,
                                                          double* __restrict__ qhat, const double* __restrict__ qcur,
                                                          double* last_q, double* last_g, double* dq, double* dg,
                                                          double* partial18, unsigned int* tickets) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int s = blockIdx.y;
  hdk_ctl* ctl = ctls + s;
  if (ctl->cond == 0) return;  // this sample's loop has ended
  const size_t n3 = 3 * (size_t)x.nv;  // ring stride: the whole batch
  const size_t i0 = 3 * (size_t)s * g.nv, i1 = i0 + 3 * (size_t)g.nv;
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
  for (size_t i = i0 + blockIdx.x * kT + threadIdx.x; i < i1; i += (size_t)gridDim.x * kT) {
    const int v = static_cast<int>(i / 3), a = static_cast<int>(i - 3 * (size_t)v);
    const int2 vf = __ldg(f.vfold + v);
    double th;
    if (vf.y > 0) {
      th = 0.0;
      for (int b = 0; b < vf.y; ++b) th += __ldg(f.part2 + 3 * ((size_t)vf.x + 256 * (size_t)b) + a);
      qhat[i] = th;
    } else {
      th = qhat[i];
    }
    const double qc = qcur[i];
    const double gv = th - qc;
    acc[2 * HDK_AA_MAX] += gv * gv;
    acc[2 * HDK_AA_MAX + 1] += th * th;
    if (push) {
      const double dqn = qc - last_q[i];
      const double dgn = gv - last_g[i];
      dq[ns * n3 + i] = dqn;
      dg[ns * n3 + i] = dgn;
#pragma unroll
      for (int j = 0; j < HDK_AA_MAX; ++j) {
        if (j < c2) {
          const int ph = (h2 + j) % m;
          const double dgj = ph == ns ? dgn : dg[ph * n3 + i];
          acc[j] += dgn * dgj;
          acc[HDK_AA_MAX + j] += dgj * gv;
        }
      }
    }
    last_q[i] = qc;
    last_g[i] = gv;
  }
  double* part = partial18 + s * kPS;
  block_partials_18(acc, part);
  __shared__ int is_last;
  if (threadIdx.x < 18) __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(tickets + s, 1u);
    is_last = t == gridDim.x - 1;
    if (is_last) tickets[s] = 0u;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  aa_solve_block(ctl, ctl, part, 0, 0, 0);
}

__global__ void __launch_bounds__(kT) k_seg_aa_mix(hdk_vtx x, hdk_segs g, hdk_ctl* ctls, const double* __restrict__ qhat,
                                                   double* qcur, double* qprev, const double* __restrict__ dq,
                                                   const double* __restrict__ dg, double* partial) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int s = blockIdx.y;
  const hdk_ctl* ctl = ctls + s;
  if (ctl->cond == 0) return;
  const size_t n3 = 3 * (size_t)x.nv;
  const size_t i0 = 3 * (size_t)s * g.nv, i1 = i0 + 3 * (size_t)g.nv;
  const int mixed = ctl->mixed, c = ctl->count, h = ctl->head, m = ctl->window;
  double gam[HDK_AA_MAX];
#pragma unroll
  for (int j = 0; j < HDK_AA_MAX; ++j) gam[j] = j < c ? ctl->gamma[j] : 0.0;
  double acc[2] = {0.0, 0.0};
  for (size_t i = i0 + blockIdx.x * kT + threadIdx.x; i < i1; i += (size_t)gridDim.x * kT) {
    const double qc = qcur[i], th = qhat[i];
    double out = qc + (th - qc);
    if (mixed) {
#pragma unroll
      for (int j = 0; j < HDK_AA_MAX; ++j)
        if (j < c) {
          const int ph = (h + j) % m;
          out -= gam[j] * (dq[ph * n3 + i] + dg[ph * n3 + i]);
        }
    }
    const double d = out - qc;
    acc[0] += d * d;
    acc[1] += qc * qc;
    qprev[i] = qc;
    qcur[i] = out;
  }
  block_partials<2>(acc, partial + s * kPS);
}

// OR over the samples of "still iterating" (thread-strided, block-wide).
__device__ __forceinline__ int seg_any_value(const hdk_ctl* ctl, int count) {
  int on = 0;
  for (int t = threadIdx.x; t < count; t += blockDim.x)
    on |= (ctl[t].cond != 0 && ctl[t].err == 0 && ctl[t].nonfinite == 0) ? 1 : 0;
  return __syncthreads_or(on);
}

__global__ void __launch_bounds__(kT) k_seg_gate(hdk_ctl* ctls, hdk_segs g, const double* pb, const double* pq,
                                                 int* any, unsigned int* ticket, cudaGraphConditionalHandle handle,
                                                 int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int s = blockIdx.x;
  hdk_ctl* ctl = ctls + s;
  __shared__ double sb[2], sq[2];
  if (ctl->cond != 0) {  // uniform per block
    fold_rb(pb + s * kPS, 2, sb);
    fold_rb(pq + s * kPS, 2, sq);
    __syncthreads();
    if (threadIdx.x == 0) {
      const double db = sb[0], bb = sb[1], dqq = sq[0], qq = sq[1];
      const int k = ctl->k;
      const double er = ctl->eps_rel, ea = ctl->eps_abs;
      const bool gate = k >= 1 && sqrt(dqq) <= er * sqrt(qq) + ea && sqrt(db) <= er * sqrt(bb) + ea;
      ctl->k = k + 1;
      ctl->iterations = k + 1;
      if (gate) ctl->converged = 1;
      ctl->cond = (!gate && k + 1 < ctl->k_max && ctl->err == 0) ? 1 : 0;
    }
  }
  __shared__ int is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    is_last = t == gridDim.x - 1;
    if (is_last) *ticket = 0u;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const int a = seg_any_value(ctls, g.count);
  if (threadIdx.x == 0) {
    *any = a;
    if (use_handle) cudaGraphSetConditional(handle, a);
  }
}

__global__ void k_seg_any(const hdk_ctl* ctls, hdk_segs g, int* any, cudaGraphConditionalHandle handle,
                          int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int a = seg_any_value(ctls, g.count);
  if (threadIdx.x == 0) {
    *any = a;
    if (use_handle) cudaGraphSetConditional(handle, a);
  }
}

__global__ void k_seg_commit(hdk_segs g, const hdk_ctl* ctl, const double* qs, double h, double* q, double* v) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const size_t per = 3 * (size_t)g.nv;
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= per * g.count || ctl[i / per].err != 0) return;
  const double sq = qs[i];
  v[i] = (sq - q[i]) / h;
  q[i] = sq;
}

__global__ void __launch_bounds__(kT) k_seg_tr_spmv(hdk_csr A, hdk_segs g, const double* __restrict__ dq,
                                                    double* partial) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int s = blockIdx.y;
  double acc[1] = {0.0};
  const int p0 = s * g.n, p1 = p0 + g.n;
  for (int p = p0 + blockIdx.x * kT + threadIdx.x; p < p1; p += gridDim.x * kT) {
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
  block_partials<1>(acc, partial + s * kPS);
}

__global__ void __launch_bounds__(kT) k_seg_tr_partials(hdk_vtx x, hdk_segs g, const double* ep, const double* es,
                                                        const double* qp, const double* qs, const double* qt,
                                                        double* partial) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int s = blockIdx.y;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int n = max(g.ne, g.nv);
  for (int il = blockIdx.x * kT + threadIdx.x; il < n; il += gridDim.x * kT) {
    if (il < g.ne) {
      acc[0] += ep[(size_t)s * g.ne + il];
      acc[1] += es[(size_t)s * g.ne + il];
    }
    const int i = s * g.nv + il;
    if (il < g.nv && x.v2p[i] >= 0) {
      const double m = x.mass[i];
      for (int a = 0; a < 3; ++a) {
        const size_t j = 3 * (size_t)i + a;
        const double d0 = qp[j] - qt[j], d1 = qs[j] - qt[j];
        acc[2] += d0 * m * d0;
        acc[3] += d1 * m * d1;
      }
    }
  }
  block_partials<4>(acc, partial + s * kPS);
}

__global__ void __launch_bounds__(kT) k_seg_tr_final(hdk_ctl* ctls, const double* pm, const double* pe,
                                                     double inv_h2) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int s = blockIdx.x;
  hdk_ctl* ctl = ctls + s;
  __shared__ double sm_[1], se[4];
  fold_rb(pm + s * kPS, 1, sm_);
  fold_rb(pe + s * kPS, 4, se);
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

__global__ void __launch_bounds__(kT) k_seg_bb_dots(int n, hdk_factor f, hdk_segs g, hdk_ctl* ctl, hdk_ctl* snap,
                                                    double* __restrict__ tp, double* __restrict__ tv,
                                                    const double* __restrict__ xp, double* last_q, double* last_g,
                                                    double* dq, double* dg, double* partial18) {
  const int s = blockIdx.y;
  bb_dots_body(n, f, ctl + s, snap + s, tp, tv, xp, last_q, last_g, dq, dg, partial18 + s * kPS, 0,
               3 * (size_t)s * g.n, 3 * (size_t)g.n);
}

__global__ void __launch_bounds__(kT) k_seg_bb_solve(hdk_ctl* ctl, const hdk_ctl* snap, const double* partial18,
                                                     AaResult* out) {
  const int s = blockIdx.x;
  bb_solve_body(ctl + s, snap + s, partial18 + s * kPS, out + s, 0, 0);
}

__global__ void __launch_bounds__(kT) k_seg_bb_mix(int n, const int* __restrict__ p2v, hdk_segs g, hdk_ctl* ctl,
                                                   const hdk_ctl* snap, const AaResult* __restrict__ res,
                                                   const double* __restrict__ tp, double* xp, double* __restrict__ xv,
                                                   const double* __restrict__ sq, const double* __restrict__ rt,
                                                   double* rx, double* last_rx, double* last_rg, double* rsq,
                                                   const double* __restrict__ seedp, double* __restrict__ rhs) {
  const int s = blockIdx.y;
  bb_mix_body(n, p2v, ctl + s, snap + s, res + s, tp, xp, xv, sq, rt, rx, last_rx, last_rg, rsq, seedp, rhs,
              3 * (size_t)s * g.n, 3 * (size_t)g.n);
}

constexpr int kSumT = 1024;
__global__ void __launch_bounds__(kSumT) k_seg_half_sqdist(hdk_segs g, const double* __restrict__ q,
                                                           const double* __restrict__ ref, double* out) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  __shared__ double sh[32];
  const size_t per = 3 * (size_t)g.nv, base = blockIdx.x * per;
  double v = 0.0;
  for (size_t i = threadIdx.x; i < per; i += kSumT) {
    const double d = q[base + i] - ref[base + i];
    v += d * d;
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = threadIdx.x < kSumT / 32 ? sh[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (threadIdx.x == 0) out[blockIdx.x] = 0.5 * v;
}

__global__ void k_seg_sum(hdk_segs g, const double* __restrict__ vec, const double* __restrict__ loss,
                          double* __restrict__ out) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    double l = 0;
    for (int s = 0; s < g.count; ++s) l += loss[s];
    out[0] = l;
  }
  if (i < g.ne) {
    double a = 0;
    for (int s = 0; s < g.count; ++s) a += vec[(size_t)s * g.ne + i];
    out[1 + i] = a;
  }
}

}  // namespace

extern "C" {

HDK_API int hdk_seg_ctl_init(hdk_ctl* ctl, const hdk_segs* g, const int* windows, double guard, int k_max,
                             double eps_rel, double eps_abs, double tol, double eps_tr, int* any, void* stream) {
  hdk::launch(k_seg_ctl_init, dim3(1), dim3(256), 0, S(stream), ctl, *g, windows, guard, k_max, eps_rel, eps_abs, tol,
              eps_tr, any);
  return last();
}
HDK_API int hdk_seg_aa_reset(hdk_ctl* ctl, const hdk_segs* g, int window, double guard, int k_max, double tol,
                             int* any, void* stream) {
  hdk::launch(k_seg_aa_reset, dim3(1), dim3(256), 0, S(stream), ctl, *g, window, guard, k_max, tol, any);
  return last();
}
HDK_API int hdk_seg_gather_rhs(const hdk_vtx* x, const hdk_segs* g, const hdk_ctl* ctl, const double* ef,
                               double inv_h2, const double* q_tilde, const double* damp, double* b_prev,
                               double* rhs_perm, double* partial, void* stream) {
  hdk::launch(k_seg_gather_rhs<false>, dim3(kRB, g->count), dim3(kT), 0, S(stream), *x, *g, ef, inv_h2, q_tilde, damp,
              b_prev, rhs_perm, partial, ctl);
  return last();
}
HDK_API int hdk_seg_gather_rhs_sorted(const hdk_vtx* x, const hdk_segs* g, const hdk_ctl* ctl, const double* efs,
                                      double inv_h2, const double* q_tilde, const double* damp, double* b_prev,
                                      double* rhs_perm, double* partial, void* stream) {
  hdk::launch(k_seg_gather_rhs<true>, dim3(kRB, g->count), dim3(kT), 0, S(stream), *x, *g, efs, inv_h2, q_tilde, damp,
              b_prev, rhs_perm, partial, ctl);
  return last();
}
HDK_API int hdk_seg_aa_dots_fused(const hdk_vtx* x, const hdk_factor* f, const hdk_segs* g, hdk_ctl* ctl,
                                  double* qhat, const double* qcur, double* last_q, double* last_g, double* dq,
                                  double* dg, double* partial18, unsigned int* tickets, void* stream) {
  hdk::launch(k_seg_aa_dots_fused, dim3(kRB, g->count), dim3(kT), 0, S(stream), *x, *f, *g, ctl, qhat, qcur, last_q,
              last_g, dq, dg, partial18, tickets);
  return last();
}
HDK_API int hdk_seg_aa_mix(const hdk_vtx* x, const hdk_segs* g, hdk_ctl* ctl, const double* qhat, double* qcur,
                           double* qprev, const double* dq, const double* dg, double* partial, void* stream) {
  hdk::launch(k_seg_aa_mix, dim3(kRB, g->count), dim3(kT), 0, S(stream), *x, *g, ctl, qhat, qcur, qprev, dq, dg,
              partial);
  return last();
}
HDK_API int hdk_seg_gate(hdk_ctl* ctl, const hdk_segs* g, const double* partial_b, const double* partial_q, int* any,
                         unsigned int* ticket, unsigned long long cond_handle, void* stream) {
  hdk::launch(k_seg_gate, dim3(g->count), dim3(kT), 0, S(stream), ctl, *g, partial_b, partial_q, any, ticket,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle ? 1 : 0);
  return last();
}
HDK_API int hdk_seg_commit(const hdk_segs* g, const hdk_ctl* ctl, const double* q_star, double h, double* q, double* v,
                           void* stream) {
  hdk::launch(k_seg_commit, dim3(nb(3LL * g->nv * g->count)), dim3(256), 0, S(stream), *g, ctl, q_star, h, q, v);
  return last();
}
HDK_API int hdk_seg_tr_model(const hdk_vtx* x, const hdk_segs* g, const hdk_csr* a_ff, const double* q_star,
                             const double* q_prev, double* dq_perm, double* partial, void* stream) {
  hdk::launch(k_tr_dq, dim3(nb(x->n)), dim3(256), 0, S(stream), *x, q_star, q_prev, dq_perm);
  hdk::launch(k_seg_tr_spmv, dim3(kRB, g->count), dim3(kT), 0, S(stream), *a_ff, *g, dq_perm, partial);
  return last();
}
HDK_API int hdk_seg_tr_select(const hdk_vtx* x, const hdk_segs* g, const double* e_prev, const double* e_star,
                              const double* q_prev, const double* q_star, const double* q_tilde, double inv_h2,
                              const double* model_partial, double* partial, hdk_ctl* ctl, void* stream) {
  hdk::launch(k_seg_tr_partials, dim3(kRB, g->count), dim3(kT), 0, S(stream), *x, *g, e_prev, e_star, q_prev, q_star,
              q_tilde, partial);
  hdk::launch(k_seg_tr_final, dim3(g->count), dim3(kT), 0, S(stream), ctl, model_partial, partial, inv_h2);
  return last();
}
HDK_API int hdk_seg_bb_dots(const hdk_factor* f, const hdk_segs* g, hdk_ctl* ctl, hdk_ctl* snap, double* t_perm,
                            double* t_full, const double* x_perm, double* last_q, double* last_g, double* dq,
                            double* dg, double* partial18, void* stream) {
  hdk::launch(k_seg_bb_dots, dim3(kRB, g->count), dim3(kT), 0, S(stream), f->n, *f, *g, ctl, snap, t_perm, t_full,
              x_perm, last_q, last_g, dq, dg, partial18);
  return last();
}
HDK_API int hdk_seg_bb_solve(hdk_ctl* ctl, const hdk_segs* g, const hdk_ctl* snap, const double* partial18,
                             void* results, void* stream) {
  hdk::launch(k_seg_bb_solve, dim3(g->count), dim3(kT), 0, S(stream), ctl, snap, partial18,
              static_cast<AaResult*>(results));
  return last();
}
HDK_API int hdk_seg_bb_mix(const hdk_factor* f, const hdk_segs* g, hdk_ctl* ctl, const hdk_ctl* snap,
                           const void* results, const double* t_perm, double* x_perm, double* x_full,
                           const double* sum_hist, const double* rt_perm, double* rx_perm, double* last_rx,
                           double* last_rg, double* rsum_hist, const double* seed_perm, double* rhs_perm,
                           void* stream) {
  hdk::launch(k_seg_bb_mix, dim3(nb(3LL * g->n), g->count), dim3(kT), 0, S(stream), f->n, f->p2v, *g, ctl, snap,
              static_cast<const AaResult*>(results), t_perm, x_perm, x_full, sum_hist, rt_perm, rx_perm, last_rx,
              last_rg, rsum_hist, seed_perm, rhs_perm);
  return last();
}
HDK_API int hdk_seg_any(const hdk_ctl* ctl, const hdk_segs* g, int* any, unsigned long long cond_handle, void* stream) {
  hdk::launch(k_seg_any, dim3(1), dim3(256), 0, S(stream), ctl, *g, any,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle ? 1 : 0);
  return last();
}
HDK_API int hdk_seg_half_sqdist(const hdk_segs* g, const double* q, const double* ref, double* out, void* stream) {
  hdk::launch(k_seg_half_sqdist, dim3(g->count), dim3(kSumT), 0, S(stream), *g, q, ref, out);
  return last();
}
HDK_API int hdk_seg_sum(const hdk_segs* g, const double* vec, const double* loss, double* out, void* stream) {
  hdk::launch(k_seg_sum, dim3(nb(g->ne > 0 ? g->ne : 1)), dim3(256), 0, S(stream), *g, vec, loss, out);
  return last();
}

}  // extern "C"
