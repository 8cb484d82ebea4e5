// Contact kernels (reference contact.cpp, forward.cpp:171-250,
// backward.cpp:227-283), device-resident end to end: detection, compaction
// and geometry (hdk_contact_setup), the scalar inverse columns and the
// Delassus matrix, the per-iteration multiplier update with its dense LDL^T
// (dense.cuh), and the adjoint's reduced multiplier system.  Counts live in
// device memory (hdk_contacts::cnt), so every kernel is launched for the
// capacities and reads the live sizes itself; the whole contact step is part
// of the forward CUDA graph.  Rows follow the reference's stacked order:
// normals, then two tangent rows per frictional contact.
//
// Arithmetic that decides contact membership and geometry (signed distance,
// normal, gap offset, tangent basis) is written with explicit round-to-
// nearest products and sums in the reference's evaluation order (no FMA
// contraction), so identical positions give identical contact rows.
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>

#include "../../include/hdk.h"
#include "dense.cuh"
#include "launch.cuh"

namespace {

using hdk::add;
using hdk::mul;
using hdk::sub;

constexpr int kSetupT = 1024;
constexpr int kNcpT = 512;
constexpr int kSmemRows = 224;  // systems up to this capacity factor in shared memory (packed lower triangle)

__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return add(add(mul(a[0], b[0]), mul(a[1], b[1])), mul(a[2], b[2]));
}

// Signed distance of x to obstacle ob (contact.cpp:39-45).
__device__ double signed_distance(const double* ob, const double* x) {
  if (ob[0] == 0.0) return sub(dot3(ob + 1, x), ob[4]);
  const double d[3] = {sub(x[0], ob[5]), sub(x[1], ob[6]), sub(x[2], ob[7])};
  return sub(__dsqrt_rn(dot3(d, d)), ob[4]);
}

// Outward normal (contact.cpp:46-52) and deterministic tangent basis (:54-66).
__device__ void normal_of(const double* ob, const double* x, double* n) {
  if (ob[0] == 0.0) {
    n[0] = ob[1];
    n[1] = ob[2];
    n[2] = ob[3];
    return;
  }
  const double d[3] = {sub(x[0], ob[5]), sub(x[1], ob[6]), sub(x[2], ob[7])};
  const double len = __dsqrt_rn(dot3(d, d));
  if (len < 1e-12) {
    n[0] = 0.0;
    n[1] = 1.0;
    n[2] = 0.0;
    return;
  }
  for (int a = 0; a < 3; ++a) n[a] = d[a] / len;
}
__device__ void cross(const double* a, const double* b, double* o) {
  o[0] = sub(mul(a[1], b[2]), mul(a[2], b[1]));
  o[1] = sub(mul(a[2], b[0]), mul(a[0], b[2]));
  o[2] = sub(mul(a[0], b[1]), mul(a[1], b[0]));
}
__device__ void tangents(const double* n, double* t1, double* t2) {
  const double a0 = fabs(n[0]), a1 = fabs(n[1]), a2 = fabs(n[2]);
  double axis[3] = {1.0, 0.0, 0.0};
  if (a1 <= a0 && a1 <= a2) {
    axis[0] = 0.0;
    axis[1] = 1.0;
  } else if (a2 <= a0 && a2 <= a1) {
    axis[0] = 0.0;
    axis[2] = 1.0;
  }
  cross(n, axis, t1);
  const double l = __dsqrt_rn(dot3(t1, t1));
  for (int a = 0; a < 3; ++a) t1[a] = t1[a] / l;
  cross(n, t1, t2);
}

// Block-wide inclusive scan of one int per thread (kSetupT threads);
// returns the inclusive prefix, *total the block sum.
__device__ int block_scan(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();  // warp_tot reuse across calls
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < kSetupT / 32 ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  *total = warp_tot[kSetupT / 32 - 1];
  return x + (w > 0 ? warp_tot[w - 1] : 0);
}

__global__ void __launch_bounds__(kSetupT) k_setup(int nv, const int* __restrict__ v2p, const double* __restrict__ q,
                                                   int no, const double* __restrict__ obs, double margin, hdk_contacts c,
                                                   hdk_ctl* ctl, cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  __shared__ int warp_tot[32];
  const long long total = static_cast<long long>(nv) * no;
  int run_c = 0, run_u = 0;
  // pass A: detection, compaction, geometry; first contact of each vertex = unique slot
  for (long long base = 0; base < total; base += kSetupT) {
    const long long i = base + threadIdx.x;
    int flag = 0, first = 0, v = 0, o = 0;
    double x[3];
    if (i < total) {
      v = static_cast<int>(i / no);
      o = static_cast<int>(i - static_cast<long long>(v) * no);
      if (v2p[v] >= 0) {
        x[0] = q[3 * (size_t)v];
        x[1] = q[3 * (size_t)v + 1];
        x[2] = q[3 * (size_t)v + 2];
        if (!(signed_distance(obs + HDK_OBSTACLE_DOUBLES * o, x) > margin)) {  // contact.cpp:131
          flag = 1;
          first = 1;
          for (int p = 0; p < o; ++p)
            if (!(signed_distance(obs + HDK_OBSTACLE_DOUBLES * p, x) > margin)) first = 0;
        }
      }
    }
    int tot;
    const int incl = block_scan(flag | (first << 16), warp_tot, &tot);
    const int excl = incl - (flag | (first << 16));
    const int ci = run_c + (excl & 0xffff);
    const int u = run_u + (incl >> 16) - 1;  // unique slot of this vertex
    if (flag && ci < c.cap_c) {
      const double* ob = obs + HDK_OBSTACLE_DOUBLES * o;
      double n[3], t1[3], t2[3];
      normal_of(ob, x, n);
      tangents(n, t1, t2);
      c.vertex[ci] = v;
      c.obstacle[ci] = o;
      for (int a = 0; a < 3; ++a) {
        c.normal[3 * ci + a] = n[a];
        c.t1[3 * ci + a] = t1[a];
        c.t2[3 * ci + a] = t2[a];
      }
      c.gap[ci] = sub(dot3(n, x), signed_distance(ob, x));
      c.mu[ci] = ob[8];
      c.row_unique[ci] = u;  // cap_k >= cap_c
    }
    if (first && u < c.cap_u) {
      c.unique_pos[u] = v2p[v];
      c.nfirst[u] = ci;
    }
    run_c += tot & 0xffff;
    run_u += tot >> 16;
  }
  __syncthreads();  // pass A's stores before B and C read them
  const int nc = run_c, nu = run_u;
  bool over = nc > c.cap_c || nu > c.cap_u || nc > c.cap_k;
  // pass B: frictional contacts in contact order
  int nf = 0;
  if (!over) {
    for (int base = 0; base < nc; base += kSetupT) {
      const int i = base + threadIdx.x;
      const int flag = (i < nc && c.mu[i] > 0.0) ? 1 : 0;
      int tot;
      const int incl = block_scan(flag, warp_tot, &tot);
      if (i < nc) {
        c.fpre[i] = nf + incl - flag;
        if (flag) c.fric[nf + incl - 1] = i;
      }
      nf += tot;
    }
  }
  const int k = nc + 2 * nf;
  over = over || k > c.cap_k;
  if (!over) {
    if (threadIdx.x == 0) {
      c.fpre[nc] = nf;
      c.nfirst[nu] = nc;
    }
    __syncthreads();
    // pass C: rows of each unique vertex (its normal rows, then its tangent rows)
    for (int i = threadIdx.x; i < nc; i += kSetupT) {
      const int u = c.row_unique[i];
      const int f0 = c.nfirst[u];
      const int off = f0 + 2 * c.fpre[f0];
      c.urow[off + (i - f0)] = i;
      if (c.mu[i] > 0.0) {
        const int f = c.fpre[i];
        const int pos = off + (c.nfirst[u + 1] - f0) + 2 * (f - c.fpre[f0]);
        c.urow[pos] = nc + 2 * f;
        c.urow[pos + 1] = nc + 2 * f + 1;
        c.row_unique[nc + 2 * f] = u;
        c.row_unique[nc + 2 * f + 1] = u;
      }
    }
    for (int u = threadIdx.x; u <= nu; u += kSetupT) c.urow_off[u] = c.nfirst[u] + 2 * c.fpre[c.nfirst[u]];
    for (int r = threadIdx.x; r < k; r += kSetupT) c.lambda[r] = 0.0;  // zero_multipliers
  }
  if (threadIdx.x == 0) {
    c.cnt[HDK_CNT_NC] = over ? 0 : nc;
    c.cnt[HDK_CNT_NF] = over ? 0 : nf;
    c.cnt[HDK_CNT_K] = over ? 0 : k;
    c.cnt[HDK_CNT_NU] = over ? 0 : nu;
    c.cnt[HDK_CNT_OVERFLOW] = over ? 1 : 0;
    c.cnt[HDK_CNT_NEED_C] = nc;
    c.cnt[HDK_CNT_NEED_K] = k;
    c.cnt[HDK_CNT_NEED_U] = nu;
    c.cnt[HDK_CNT_SPIKE] = 0;
    const int run = (!over && nu > 0) ? 1 : 0;
    c.cnt[HDK_CNT_SPIKE_COND] = run;
    if (over) atomicCAS(&ctl->err, 0, HDK_ERR_CAPACITY);
    if (use_handle) cudaGraphSetConditional(handle, run);
  }
}

// Inverse-column loop: spikes of unique slots [u0, u0 + 3) on the three axes.
__global__ void k_spikes(hdk_contacts c, double* rhs_perm) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= c.n) return;
  const int u0 = c.cnt[HDK_CNT_SPIKE], cnt = min(3, c.cnt[HDK_CNT_NU] - u0);
  for (int a = 0; a < 3; ++a) rhs_perm[3 * (size_t)p + a] = (a < cnt && c.unique_pos[u0 + a] == p) ? 1.0 : 0.0;
}
__global__ void k_unspike(hdk_contacts c, const double* x_perm) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= c.n) return;
  const int u0 = c.cnt[HDK_CNT_SPIKE], cnt = min(3, c.cnt[HDK_CNT_NU] - u0);
  for (int a = 0; a < cnt; ++a) c.U[(size_t)(u0 + a) * c.n + p] = x_perm[3 * (size_t)p + a];
}
__global__ void k_spike_next(hdk_contacts c, cudaGraphConditionalHandle handle, int use_handle) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int next = c.cnt[HDK_CNT_SPIKE] + 3;
  const int run = next < c.cnt[HDK_CNT_NU] ? 1 : 0;
  c.cnt[HDK_CNT_SPIKE] = next;
  c.cnt[HDK_CNT_SPIKE_COND] = run;
  if (use_handle) cudaGraphSetConditional(handle, run);
}

// Row direction and vertex of stacked row r.
__device__ __forceinline__ void row_of(const hdk_contacts& c, int nc, int r, int& v, const double*& d) {
  if (r < nc) {
    v = c.vertex[r];
    d = c.normal + 3 * r;
  } else {
    const int ci = c.fric[(r - nc) >> 1];
    v = c.vertex[ci];
    d = ((r - nc) & 1) ? c.t2 + 3 * ci : c.t1 + 3 * ci;
  }
}

// W(r, s) = (d_r . d_s) gram(u_r, u_s), one triangle mirrored (factor.cpp:418-422).
__global__ void k_delassus(hdk_contacts c) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int k = c.cnt[HDK_CNT_K], nc = c.cnt[HDK_CNT_NC];
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (idx >= (size_t)k * k) return;
  const int s = static_cast<int>(idx / k), r = static_cast<int>(idx % k);
  int vr, vs;
  const double *dr, *ds;
  row_of(c, nc, r, vr, dr);
  row_of(c, nc, s, vs, ds);
  const int ur = c.row_unique[r], us = c.row_unique[s];
  const int ua = ur < us ? ur : us, ub = ur < us ? us : ur;
  c.W[idx] = mul(dot3(dr, ds), c.U[(size_t)ua * c.n + c.unique_pos[ub]]);
}
// r_n = h^2 W_nn, r_f = h^2 (W_t1t1 + W_t2t2)/2 (forward.cpp:183-192).
__global__ void k_rdiag(hdk_contacts c, double h) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int nc = c.cnt[HDK_CNT_NC], nf = c.cnt[HDK_CNT_NF], k = c.cnt[HDK_CNT_K];
  const double h2 = mul(h, h);
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    c.r_n[i] = mul(h2, c.W[(size_t)i * k + i]);
    c.r_f[i] = 0.0;
  }
  __syncthreads();
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    const int fr = nc + 2 * f;
    c.r_f[c.fric[f]] = mul(mul(h2, 0.5), add(c.W[(size_t)fr * k + fr], c.W[(size_t)(fr + 1) * k + fr + 1]));
  }
}

// Fischer-Burmeister NCP weights (ncp_weights, contact.cpp:151-158).
__device__ __forceinline__ void ncp(double delta, double r, double lambda, double& om, double& e) {
  const double root = __dsqrt_rn(add(mul(delta, delta), mul(mul(mul(r, r), lambda), lambda)));
  if (root == 0.0) {  // active-branch limit at the origin
    om = 1.0;
    e = r;
    return;
  }
  om = sub(1.0, delta / root);
  e = mul(sub(1.0, mul(r, lambda) / root), r);
}

// Weights of every row (contact_weights, contact.cpp:160-196); thread-strided.
__device__ void weights_rows(const hdk_contacts& c, int nc, int nf, const double* q, const double* qt,
                             const double* lambda, double* om_out, double* e_out) {
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const int v = c.vertex[i];
    const double delta = sub(dot3(c.normal + 3 * i, q + 3 * (size_t)v), c.gap[i]);
    double om, e;
    ncp(delta, c.r_n[i], lambda[i], om, e);
    om_out[i] = om;
    e_out[i] = e;
  }
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    const int ci = c.fric[f];
    const int v = c.vertex[ci];
    const double d[3] = {sub(q[3 * (size_t)v], qt[3 * (size_t)v]), sub(q[3 * (size_t)v + 1], qt[3 * (size_t)v + 1]),
                         sub(q[3 * (size_t)v + 2], qt[3 * (size_t)v + 2])};
    const double slip = hdk::libm_hypot(dot3(c.t1 + 3 * ci, d), dot3(c.t2 + 3 * ci, d));
    const int row = nc + 2 * f;
    const double lam_f = hdk::libm_hypot(lambda[row], lambda[row + 1]);
    const double slack = sub(mul(c.mu[ci], lambda[ci]), lam_f);
    double om, e;
    ncp(slip, c.r_f[ci], slack, om, e);
    om_out[row] = om_out[row + 1] = om;
    e_out[row] = e_out[row + 1] = e;
  }
}

__global__ void k_weights(hdk_contacts c, const double* q, const double* qt) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  weights_rows(c, c.cnt[HDK_CNT_NC], c.cnt[HDK_CNT_NF], q, qt, c.lambda, c.omega, c.e_diag);
}

// Shared-memory layout of the single-CTA system kernels.
struct SysSmem {
  double *M, *om, *ed, *wl, *rhs, *diag;
  int *perm, *byval, *gsz, *pos, *at;
};
__device__ SysSmem carve(double* base, int cap, double* Mg) {
  SysSmem s;
  double* p = base;
  if (Mg) {
    s.M = Mg;
  } else {
    s.M = p;
    p += hdk::Packed::doubles(cap);
  }
  s.om = p; p += cap;
  s.ed = p; p += cap;
  s.wl = p; p += cap;
  s.rhs = p; p += cap;
  s.diag = p; p += cap;
  int* ip = reinterpret_cast<int*>(p);
  s.perm = ip; ip += cap;
  s.byval = ip; ip += cap;
  s.gsz = ip; ip += cap;
  s.pos = ip; ip += cap;
  s.at = ip;
  return s;
}
size_t smem_bytes(int cap, bool with_matrix) {
  return (with_matrix ? hdk::Packed::doubles(cap) * 8 : 0) + (size_t)cap * (5 * 8 + 5 * 4);
}

// Multiplier update of one PD iteration (forward.cpp:226-235).
__global__ void __launch_bounds__(kNcpT) k_ncp(hdk_contacts c, const double* __restrict__ qc,
                                               const double* __restrict__ qt, const double* __restrict__ q0,
                                               double* Mg, hdk_ctl* ctl, hdk_contact_trace tr) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  extern __shared__ double dsm[];
  const int nc = c.cnt[HDK_CNT_NC], nf = c.cnt[HDK_CNT_NF], k = c.cnt[HDK_CNT_K], nu = c.cnt[HDK_CNT_NU];
  if (k == 0) return;
  SysSmem s = carve(dsm, c.cap_k, Mg);
  __shared__ double lift_sh;
  // weights at q_cur with the current multipliers
  weights_rows(c, nc, nf, qc, qt, c.lambda, s.om, s.ed);
  __syncthreads();
  for (int r = threadIdx.x; r < k; r += kNcpT) {
    c.omega[r] = s.om[r];
    c.e_diag[r] = s.ed[r];
    s.wl[r] = mul(s.om[r], c.lambda[r]);
    // diagonal of Omega W Omega + E (contact.cpp:242-246)
    s.diag[r] = add(mul(mul(s.om[r], c.W[(size_t)r * k + r]), s.om[r]), s.ed[r]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr_sum = 0.0;
    for (int r = 0; r < k; ++r) tr_sum = add(tr_sum, s.diag[r]);
    lift_sh = mul(1e-10, tr_sum) / k;
  }
  __syncthreads();
  const double lift = lift_sh;
  for (int r = threadIdx.x; r < k; r += kNcpT) {
    s.diag[r] = add(s.diag[r], lift);
    // rhs = h_vec - omega o J q_mid, J q_mid = J q0 + W (omega o lambda)
    int v;
    const double* d;
    row_of(c, nc, r, v, d);
    double jq = dot3(d, q0 + 3 * (size_t)v);
    for (int t = 0; t < k; ++t) jq = add(jq, mul(c.W[(size_t)t * k + r], s.wl[t]));
    const double hv = r < nc ? mul(s.om[r], c.gap[r]) : mul(s.om[r], dot3(d, qt + 3 * (size_t)v));
    s.rhs[r] = sub(hv, mul(s.om[r], jq));
  }
  __syncthreads();
  int bad = hdk::ldlt_pivots(k, s.diag, s.perm, s.byval, s.gsz, s.pos, s.at);
  const hdk::Packed Mp{s.M, k};
  if (!bad) {
    // P M P^T, lower triangle, and the permuted right-hand side
    for (int j = threadIdx.x >> 5; j < k; j += kNcpT / 32) {  // column j by one warp
      const int q = s.perm[j];
      const double* wq = c.W + (size_t)q * k;
      for (int i = j + (threadIdx.x & 31); i < k; i += 32) {
        const int r = s.perm[i];
        double m = mul(mul(s.om[r], wq[r]), s.om[q]);
        if (i == j) m = add(add(m, s.ed[r]), lift);
        Mp(i, j) = m;
      }
    }
    for (int i = threadIdx.x; i < k; i += kNcpT) s.wl[i] = s.rhs[s.perm[i]];
    __syncthreads();
    bad = hdk::ldlt_factor(Mp);
    if (!bad) hdk::ldlt_substitute(Mp, s.wl);
  }
  // lambda + step, clamp, cone projection (project_multipliers, contact.cpp:218-235)
  __shared__ int nonfinite;
  if (threadIdx.x == 0) nonfinite = bad;
  __syncthreads();
  const int it = ctl->k;
  const bool rec = tr.clamp && it < tr.cap;
  if (!nonfinite) {
    for (int i = threadIdx.x; i < k; i += kNcpT) {
      const double step = s.wl[i];
      if (!isfinite(step)) nonfinite = 1;
      s.rhs[s.perm[i]] = add(c.lambda[s.perm[i]], step);
    }
  }
  __syncthreads();
  if (nonfinite) {
    if (threadIdx.x == 0) atomicCAS(&ctl->err, 0, 9);
    return;
  }
  for (int i = threadIdx.x; i < nc; i += kNcpT) {
    const double l = s.rhs[i];
    if (rec) tr.clamp[(size_t)it * c.cap_c + i] = l;  // clamped iff < 0
    s.rhs[i] = 0.0 < l ? l : 0.0;  // std::max(0.0, l)
  }
  __syncthreads();
  for (int f = threadIdx.x; f < nf; f += kNcpT) {
    const int ci = c.fric[f];
    const int row = nc + 2 * f;
    const double bound = mul(c.mu[ci], s.rhs[ci]);
    const double lf = hdk::libm_hypot(s.rhs[row], s.rhs[row + 1]);
    const bool out = lf > bound;
    // trace: projected onto a cone of positive radius iff > 0 (with bound == 0
    // the pair becomes 0 whether or not it was already 0: not a decision)
    if (rec) tr.cone[(size_t)it * c.cap_c + f] = bound > 0 ? (lf - bound) / bound : -1.0;
    if (out) {
      const double sc = bound > 0 ? bound / lf : 0.0;
      s.rhs[row] = mul(s.rhs[row], sc);
      s.rhs[row + 1] = mul(s.rhs[row + 1], sc);
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < k; r += kNcpT) c.lambda[r] = s.rhs[r];
  // g_u = sum over the rows of unique vertex u of (omega lambda) d
  for (int u = threadIdx.x; u < nu; u += kNcpT) {
    double g0 = 0.0, g1 = 0.0, g2 = 0.0;
    for (int j = c.urow_off[u]; j < c.urow_off[u + 1]; ++j) {
      const int r = c.urow[j];
      int v;
      const double* d;
      row_of(c, nc, r, v, d);
      const double coef = mul(s.om[r], s.rhs[r]);
      g0 = add(g0, mul(coef, d[0]));
      g1 = add(g1, mul(coef, d[1]));
      g2 = add(g2, mul(coef, d[2]));
    }
    c.g[3 * u] = g0;
    c.g[3 * u + 1] = g1;
    c.g[3 * u + 2] = g2;
  }
}

// out[v] = q0[v] + sum_u U[p(v), u] g_u on free vertices.
__global__ void k_corrected(hdk_contacts c, const int* __restrict__ p2v, const double* __restrict__ q0, double* out) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= c.n) return;
  const int nu = c.cnt[HDK_CNT_NU];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  const double* up = c.U + p;
  int u = 0;
  for (; u + 8 <= nu; u += 8) {  // eight independent column loads in flight, sums in u order
    double w[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) w[t] = up[(size_t)(u + t) * c.n];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      s0 = add(s0, mul(w[t], c.g[3 * (u + t)]));
      s1 = add(s1, mul(w[t], c.g[3 * (u + t) + 1]));
      s2 = add(s2, mul(w[t], c.g[3 * (u + t) + 2]));
    }
  }
  for (; u < nu; ++u) {
    const double w = up[(size_t)u * c.n];
    s0 = add(s0, mul(w, c.g[3 * u]));
    s1 = add(s1, mul(w, c.g[3 * u + 1]));
    s2 = add(s2, mul(w, c.g[3 * u + 2]));
  }
  const int v = p2v[p];
  out[3 * (size_t)v] = add(q0[3 * (size_t)v], s0);
  out[3 * (size_t)v + 1] = add(q0[3 * (size_t)v + 1], s1);
  out[3 * (size_t)v + 2] = add(q0[3 * (size_t)v + 2], s2);
}

// Reduced adjoint multiplier system (backward.cpp:240-262) and its solve.
__global__ void __launch_bounds__(kNcpT) k_reduced(hdk_contacts c, const double* __restrict__ X, size_t ldx,
                                                   const double* __restrict__ z0, double* Mg, int* err) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  extern __shared__ double dsm[];
  const int nc = c.cnt[HDK_CNT_NC], k = c.cnt[HDK_CNT_K];
  if (k == 0) return;
  SysSmem s = carve(dsm, c.cap_k, Mg);
  __shared__ double lift_sh;
  auto wt = [&](int d, int col) {  // d_d . X_col[v_d]
    int v;
    const double* dir;
    row_of(c, nc, d, v, dir);
    return dot3(dir, X + (size_t)col * ldx + 3 * (size_t)v);
  };
  for (int r = threadIdx.x; r < k; r += kNcpT) {
    const double om = c.omega[r];
    const double w = wt(r, r);
    const double sym = mul(0.5, add(w, w));
    s.diag[r] = add(mul(mul(om, sym), om), c.e_diag[r]);
    int v;
    const double* d;
    row_of(c, nc, r, v, d);
    s.rhs[r] = mul(om, dot3(d, z0 + 3 * (size_t)v));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr_sum = 0.0;
    for (int r = 0; r < k; ++r) tr_sum = add(tr_sum, s.diag[r]);
    lift_sh = mul(1e-10, tr_sum) / k;
  }
  __syncthreads();
  const double lift = lift_sh;
  for (int r = threadIdx.x; r < k; r += kNcpT) s.diag[r] = add(s.diag[r], lift);
  __syncthreads();
  int bad = hdk::ldlt_pivots(k, s.diag, s.perm, s.byval, s.gsz, s.pos, s.at);
  const hdk::Packed Mp{s.M, k};
  if (!bad) {
    for (int t = threadIdx.x; t < k * k; t += kNcpT) {  // once per backward frame
      const int i = t % k, j = t / k;
      if (i < j) continue;
      const int r = s.perm[i], q = s.perm[j];
      const double sym = mul(0.5, add(wt(r, q), wt(q, r)));
      double m = mul(mul(c.omega[r], sym), c.omega[q]);
      if (i == j) m = add(add(m, c.e_diag[r]), lift);
      Mp(i, j) = m;
    }
    for (int i = threadIdx.x; i < k; i += kNcpT) s.wl[i] = s.rhs[s.perm[i]];
    __syncthreads();
    bad = hdk::ldlt_factor(Mp);
    if (!bad) hdk::ldlt_substitute(Mp, s.wl);
  }
  __shared__ int nonfinite;
  if (threadIdx.x == 0) nonfinite = bad;
  __syncthreads();
  if (!nonfinite)
    for (int i = threadIdx.x; i < k; i += kNcpT) {
      if (!isfinite(s.wl[i])) nonfinite = 1;
      c.y[s.perm[i]] = s.wl[i];
    }
  __syncthreads();
  if (nonfinite && threadIdx.x == 0) atomicCAS(err, 0, 10);  // AdjointDiverged (backward.cpp:262)
}

// mu = z0 - sum_c (omega_c y_c) X_c (backward.cpp:231-234).
__global__ void k_combine(hdk_contacts c, int n3, const double* __restrict__ z0, const double* __restrict__ X,
                          size_t ldx, double* mu) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const int k = c.cnt[HDK_CNT_K];
  double s = z0[i];
  for (int col = 0; col < k; ++col) s = sub(s, mul(mul(c.omega[col], c.y[col]), X[(size_t)col * ldx + i]));
  mu[i] = s;
}

// Column right-hand side e_v d_row (full) and warm start a_row = U[:, u] d_row.
__global__ void k_column_init(hdk_contacts c, int row, int nv, const int* v2p, double* rhs, double* x0) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int nc = c.cnt[HDK_CNT_NC];
  row = min(row, c.cnt[HDK_CNT_K] - 1);
  int vr;
  const double* d;
  row_of(c, nc, row, vr, d);
  const int p = v2p[v];
  const double u = p >= 0 ? c.U[(size_t)c.row_unique[row] * c.n + p] : 0.0;
  for (int a = 0; a < 3; ++a) {
    rhs[3 * v + a] = v == vr ? d[a] : 0.0;
    x0[3 * v + a] = mul(u, d[a]);
  }
}

// Friction rows push back into dL/dq_t (backward.cpp:342-356), in row order.
__global__ void k_friction_pushback(hdk_contacts c, double* dl_dq) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int nc = c.cnt[HDK_CNT_NC], nf = c.cnt[HDK_CNT_NF];
  for (int f = 0; f < nf; ++f)
    for (int t = 0; t < 2; ++t) {
      const int row = nc + 2 * f + t;
      int v;
      const double* d;
      row_of(c, nc, row, v, d);
      const double w = mul(c.omega[row], c.y[row]);
      for (int a = 0; a < 3; ++a) dl_dq[3 * v + a] = add(dl_dq[3 * v + a], mul(w, d[a]));
    }
}

__global__ void k_test_hypot(const double* x, const double* y, double* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = hdk::libm_hypot(x[i], y[i]);
}

inline int nb(long long n) { return static_cast<int>((n + 255) / 256); }
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
inline int last() { return static_cast<int>(cudaGetLastError()); }
inline size_t align256(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }

template <typename... KArgs, typename... Args>
int launch_sys(void (*kernel)(KArgs...), int cap_k, bool global_matrix, cudaStream_t st, Args&&... args) {
  const size_t sm = smem_bytes(cap_k, !global_matrix);
  if (sm > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  hdk::launch(kernel, dim3(1), dim3(kNcpT), sm, st, args...);
  return last();
}

}  // namespace

extern "C" {

HDK_API size_t hdk_contact_block_bytes(int cap_c, int cap_k, int cap_u, int n) {
  size_t b = align256(HDK_CNT_INTS * sizeof(int));
  b += align256(sizeof(int) * cap_c) * 2;                       // vertex, obstacle
  b += align256(sizeof(double) * 3 * cap_c) * 3;                // normal, t1, t2
  b += align256(sizeof(double) * cap_c) * 4;                    // gap, mu, r_n, r_f
  b += align256(sizeof(int) * cap_c) + align256(sizeof(int) * (cap_c + 1));  // fric, fpre
  b += align256(sizeof(int) * cap_k) * 2;                       // row_unique, urow
  b += align256(sizeof(int) * (cap_u + 1)) * 2 + align256(sizeof(int) * cap_u);  // urow_off, nfirst, unique_pos
  b += align256(sizeof(double) * static_cast<size_t>(n) * cap_u);  // U
  b += align256(sizeof(double) * static_cast<size_t>(cap_k) * cap_k);  // W
  b += align256(sizeof(double) * cap_k) * 4;                    // lambda, omega, e_diag, y
  b += align256(sizeof(double) * 3 * cap_u);                    // g
  return b;
}

HDK_API void hdk_contact_block_layout(void* base, int cap_c, int cap_k, int cap_u, int n, hdk_contacts* c) {
  char* p = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += align256(bytes);
    return static_cast<void*>(r);
  };
  c->cap_c = cap_c;
  c->cap_k = cap_k;
  c->cap_u = cap_u;
  c->n = n;
  c->cnt = static_cast<int*>(take(HDK_CNT_INTS * sizeof(int)));
  c->vertex = static_cast<int*>(take(sizeof(int) * cap_c));
  c->obstacle = static_cast<int*>(take(sizeof(int) * cap_c));
  c->normal = static_cast<double*>(take(sizeof(double) * 3 * cap_c));
  c->t1 = static_cast<double*>(take(sizeof(double) * 3 * cap_c));
  c->t2 = static_cast<double*>(take(sizeof(double) * 3 * cap_c));
  c->gap = static_cast<double*>(take(sizeof(double) * cap_c));
  c->mu = static_cast<double*>(take(sizeof(double) * cap_c));
  c->r_n = static_cast<double*>(take(sizeof(double) * cap_c));
  c->r_f = static_cast<double*>(take(sizeof(double) * cap_c));
  c->fric = static_cast<int*>(take(sizeof(int) * cap_c));
  c->fpre = static_cast<int*>(take(sizeof(int) * (cap_c + 1)));
  c->row_unique = static_cast<int*>(take(sizeof(int) * cap_k));
  c->urow = static_cast<int*>(take(sizeof(int) * cap_k));
  c->urow_off = static_cast<int*>(take(sizeof(int) * (cap_u + 1)));
  c->nfirst = static_cast<int*>(take(sizeof(int) * (cap_u + 1)));
  c->unique_pos = static_cast<int*>(take(sizeof(int) * cap_u));
  c->U = static_cast<double*>(take(sizeof(double) * static_cast<size_t>(n) * cap_u));
  c->W = static_cast<double*>(take(sizeof(double) * static_cast<size_t>(cap_k) * cap_k));
  c->lambda = static_cast<double*>(take(sizeof(double) * cap_k));
  c->omega = static_cast<double*>(take(sizeof(double) * cap_k));
  c->e_diag = static_cast<double*>(take(sizeof(double) * cap_k));
  c->y = static_cast<double*>(take(sizeof(double) * cap_k));
  c->g = static_cast<double*>(take(sizeof(double) * 3 * cap_u));
}

HDK_API int hdk_contact_setup(int nv, const int* v2p, const double* q, int n_obstacles, const double* obstacles,
                              double margin, const hdk_contacts* c, hdk_ctl* ctl, unsigned long long cond_handle,
                              void* stream) {
  hdk::launch(k_setup, dim3(1), dim3(kSetupT), 0, S(stream), nv, v2p, q, n_obstacles, obstacles, margin, *c, ctl,
              static_cast<cudaGraphConditionalHandle>(cond_handle), cond_handle != 0ULL ? 1 : 0);
  return last();
}

HDK_API int hdk_contact_spikes(const hdk_contacts* c, double* rhs_perm, void* stream) {
  hdk::launch(k_spikes, dim3(nb(c->n)), dim3(256), 0, S(stream), *c, rhs_perm);
  return last();
}

HDK_API int hdk_contact_unspike(const hdk_contacts* c, const double* x_perm, unsigned long long cond_handle,
                                void* stream) {
  hdk::launch(k_unspike, dim3(nb(c->n)), dim3(256), 0, S(stream), *c, x_perm);
  hdk::launch(k_spike_next, dim3(1), dim3(32), 0, S(stream), *c, static_cast<cudaGraphConditionalHandle>(cond_handle),
              cond_handle != 0ULL ? 1 : 0);
  return last();
}

HDK_API int hdk_contact_delassus(const hdk_contacts* c, double h, void* stream) {
  hdk::launch(k_delassus, dim3(nb(static_cast<long long>(c->cap_k) * c->cap_k)), dim3(256), 0, S(stream), *c);
  hdk::launch(k_rdiag, dim3(1), dim3(256), 0, S(stream), *c, h);
  return last();
}

HDK_API int hdk_contact_weights(const hdk_contacts* c, const double* q, const double* q_t, void* stream) {
  hdk::launch(k_weights, dim3(1), dim3(256), 0, S(stream), *c, q, q_t);
  return last();
}

HDK_API int hdk_contact_smem_rows(void) { return kSmemRows; }

HDK_API int hdk_test_hypot(const double* x, const double* y, double* out, int n, void* stream) {
  k_test_hypot<<<nb(n), 256, 0, S(stream)>>>(x, y, out, n);
  return last();
}

HDK_API size_t hdk_contact_scratch_doubles(int cap_k) {
  return cap_k > kSmemRows ? hdk::Packed::doubles(cap_k) : 0;
}

HDK_API int hdk_contact_ncp(const hdk_contacts* c, const double* q_cur, const double* q_t, const double* q0,
                            double* M_scratch, hdk_ctl* ctl, const hdk_contact_trace* trace, void* stream) {
  const bool global = c->cap_k > kSmemRows;
  if (global && !M_scratch) return static_cast<int>(cudaErrorInvalidValue);
  hdk_contact_trace tr = trace ? *trace : hdk_contact_trace{nullptr, nullptr, 0};
  return launch_sys(k_ncp, c->cap_k, global, S(stream), *c, q_cur, q_t, q0, global ? M_scratch : nullptr, ctl, tr);
}

HDK_API int hdk_contact_correct(const hdk_contacts* c, const int* p2v, const double* q0, double* out, void* stream) {
  hdk::launch(k_corrected, dim3(nb(c->n)), dim3(256), 0, S(stream), *c, p2v, q0, out);
  return last();
}

HDK_API int hdk_contact_reduced(const hdk_contacts* c, const double* X, size_t ldx, const double* z0,
                                double* M_scratch, int* err, void* stream) {
  const bool global = c->cap_k > kSmemRows;
  if (global && !M_scratch) return static_cast<int>(cudaErrorInvalidValue);
  return launch_sys(k_reduced, c->cap_k, global, S(stream), *c, X, ldx, z0, global ? M_scratch : nullptr, err);
}

HDK_API int hdk_contact_combine(const hdk_contacts* c, int n3, const double* z0, const double* X, size_t ldx,
                                double* mu, void* stream) {
  hdk::launch(k_combine, dim3(nb(n3)), dim3(256), 0, S(stream), *c, n3, z0, X, ldx, mu);
  return last();
}

HDK_API int hdk_contact_column_init(const hdk_contacts* c, int row, int nv, const int* v2p, double* rhs, double* x0,
                                    void* stream) {
  hdk::launch(k_column_init, dim3(nb(nv)), dim3(256), 0, S(stream), *c, row, nv, v2p, rhs, x0);
  return last();
}

HDK_API int hdk_contact_friction_pushback(const hdk_contacts* c, double* dl_dq, void* stream) {
  hdk::launch(k_friction_pushback, dim3(1), dim3(32), 0, S(stream), *c, dl_dq);
  return last();
}

}  // extern "C"
