// Element-parallel kernels: one thread per tetrahedron, all 3x3 algebra in
// registers, structure-of-arrays element data (coalesced per field).
//
//   k_local        local_solve + element part of pd_rhs   (forward.cpp:70-117)
//                  [+ projection cache for the adjoint,   forward.cpp:252-267]
//   k_energy       primal_energy element terms            (backward.cpp:23-73)
//   k_differential tr_blend + prox differentials           (localstep.cpp:276-423,
//                  compact hat-space form, 30 doubles      backward.cpp:117-143)
//   k_bapply       matrix-free B x = sum_e V G^T (w dP/dF) G x (backward.cpp:144-163)
//   k_route_elem   dL/dw_e, dL/dE_e and the damping part of route_gradients
//                  (backward.cpp:286-394)
//   k_damp_elem    element part of damping_rhs            (forward.cpp:119-138)
//
// Element forces are written per (element, local vertex) and summed per
// vertex by a fixed-order gather (vec.cu) — no fp64 atomics, so results are
// bitwise reproducible (the reference's parallel_for contract, common.hpp:51-55).
#include <cuda_runtime.h>

#include <cstdlib>

#include "../../include/hdk.h"
#include "launch.cuh"

HDK_TRACE_TU(local)
#include "dmath.cuh"

using namespace hdk;

namespace {

struct ElemGeom {
  int v[4];
  double b[9];  // Dm^{-1} row-major
};

__device__ __forceinline__ ElemGeom load_geom(const hdk_mesh& m, int e) {
  ElemGeom g;
  const int4 t = reinterpret_cast<const int4*>(m.elem)[e];
  g.v[0] = t.x; g.v[1] = t.y; g.v[2] = t.z; g.v[3] = t.w;
#pragma unroll
  for (int k = 0; k < 9; ++k) g.b[k] = __ldg(m.bm + (size_t)k * m.ne + e);
  return g;
}

// F = [x1-x0, x2-x0, x3-x0] Dm^{-1}  (== sum_i x_i g_i^T, mesh.cpp:142-151)
__device__ __forceinline__ M3 def_grad(const ElemGeom& g, const double* __restrict__ q) {
  double x[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int a = 0; a < 3; ++a) x[i][a] = __ldg(q + 3 * (size_t)g.v[i] + a);
  M3 f;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const double d0 = x[1][r] - x[0][r], d1 = x[2][r] - x[0][r], d2 = x[3][r] - x[0][r];
#pragma unroll
    for (int c = 0; c < 3; ++c) f(r, c) = d0 * g.b[c] + d1 * g.b[3 + c] + d2 * g.b[6 + c];
  }
  return f;
}

// f_i = P g_i for the four nodes (V G^T vec(P) with V folded into P).
__device__ __forceinline__ void write_force(const ElemGeom& g, const M3& p, double* __restrict__ ef, int e) {
  double f[4][3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int k = 0; k < 3; ++k) f[k + 1][r] = p(r, 0) * g.b[3 * k] + p(r, 1) * g.b[3 * k + 1] + p(r, 2) * g.b[3 * k + 2];
    f[0][r] = -(f[1][r] + f[2][r] + f[3][r]);
  }
  double2* out = reinterpret_cast<double2*>(ef + 12 * (size_t)e);
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int i0 = 2 * k, i1 = 2 * k + 1;
    out[k] = make_double2(f[i0 / 3][i0 % 3], f[i1 / 3][i1 % 3]);
  }
}

__device__ __forceinline__ void write_force_at(const ElemGeom& g, const M3& p, double* __restrict__ efs, const int4 pos) {
  double f[4][3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int k = 0; k < 3; ++k) f[k + 1][r] = p(r, 0) * g.b[3 * k] + p(r, 1) * g.b[3 * k + 1] + p(r, 2) * g.b[3 * k + 2];
    f[0][r] = -(f[1][r] + f[2][r] + f[3][r]);
  }
  const int ps[4] = {pos.x, pos.y, pos.z, pos.w};
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (ps[k] >= 0) {
      double* o = efs + 3 * (size_t)ps[k];
      o[0] = f[k][0];
      o[1] = f[k][1];
      o[2] = f[k][2];
    }
}

// Same forces, each corner's three components stored at its slot of the
// elimination-order incidence list (corner_pos[4 e + k], -1 for fixed
// vertices), so the per-vertex gather reads one contiguous range.
__device__ __forceinline__ void write_force_sorted(const ElemGeom& g, const M3& p, double* __restrict__ efs,
                                                   const int* __restrict__ corner_pos, int e) {
  double f[4][3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int k = 0; k < 3; ++k) f[k + 1][r] = p(r, 0) * g.b[3 * k] + p(r, 1) * g.b[3 * k + 1] + p(r, 2) * g.b[3 * k + 2];
    f[0][r] = -(f[1][r] + f[2][r] + f[3][r]);
  }
  const int4 pos = __ldg(reinterpret_cast<const int4*>(corner_pos) + e);
  const int ps[4] = {pos.x, pos.y, pos.z, pos.w};
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (ps[k] >= 0) {
      double* o = efs + 3 * (size_t)ps[k];
      o[0] = f[k][0];
      o[1] = f[k][1];
      o[2] = f[k][2];
    }
}

// Prox means of element e: the material's scalars, or its sample's in a
// segmented batch (hdk_material::seg_means).
struct Means {
  double mu, lambda, k;
};
__device__ __forceinline__ Means means_of(const hdk_material& mat, int e) {
  if (!mat.seg_means) return Means{mat.mu_bar, mat.lambda_bar, mat.k_bar};
  const double* p = mat.seg_means + 3 * (e / mat.seg_ne);
  return Means{__ldg(p), __ldg(p + 1), __ldg(p + 2)};
}

__device__ __forceinline__ void set_err(int* err, int code) {
  if (err) atomicCAS(err, 0, code);
}

// Projection of one element.  Returns false on ProxDiverged.  For corotated
// materials `s` receives the volume/barrier target stretches (the rotation
// target has unit stretches).
__device__ __forceinline__ bool project(const hdk_material& mat, int e, const V3& sf, V3& s) {
  int it = 0;
  if (mat.kind == 1) {
    const Means mb = means_of(mat, e);
    const StretchNH den{mb.mu, mb.lambda};
    return newton_stretch(sf, mb.k, den, s, it);
  }
  if (mat.barrier) {
    const double mu = mat.mu_e[e], la = mat.lambda_e[e];
    const StretchBarrier den{mu, la};
    return newton_stretch(sf, 2.0 * mu + la, den, s, it);
  }
  return volume_stretch(sf, s);
}

// ctl (a segmented batch's per-sample control blocks, or NULL): an element
// of a sample whose loop has ended is skipped — its iterate no longer
// changes, so its projection and forces would be rewritten unchanged.
__global__ void __launch_bounds__(128) k_local(hdk_mesh m, hdk_material mat, const double* __restrict__ q,
                                                double* __restrict__ ef, double* __restrict__ cache, int* err,
                                                const hdk_ctl* ctl, const int* __restrict__ corner_vpos) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.ne) return;
  if (ctl && ctl[e / mat.seg_ne].cond == 0) return;
  const ElemGeom g = load_geom(m, e);
  const M3 f = def_grad(g, q);
  M3 u, v;
  V3 sf;
  signed_svd(f, u, sf, v);
  V3 s;
  if (!project(mat, e, sf, s)) set_err(err, 6);
  M3 p;
  if (mat.kind == 1) {
    const double w = mat.w1[e];
    p = recompose(u, v3(w * s[0], w * s[1], w * s[2]), v);
  } else {
    const double wr = mat.w1[e], wv = mat.w2[e];
    p = recompose(u, v3(wr + wv * s[0], wr + wv * s[1], wr + wv * s[2]), v);
  }
  // corner_vpos: each corner's force at its slot of the vertex-ordered
  // incidence list (the gather then reads contiguous ranges)
  if (corner_vpos) write_force_sorted(g, p, ef, corner_vpos, e);
  else write_force(g, p, ef, e);
  if (cache) {
    const size_t ne = m.ne;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      cache[i * ne + e] = s[i];
      cache[(3 + i) * ne + e] = sf[i];
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      cache[(6 + i) * ne + e] = u.m[i];
      cache[(15 + i) * ne + e] = v.m[i];
    }
  }
}

// V_e times the model density at the element's projection (backward.cpp:23-45);
// flags NonPositiveJacobian / ProxDiverged (tr_select_tau maps both to rho = inf).
// blockIdx.y selects one of two (q, energy) pairs: both TR energies of a
// backward frame in one launch (q2/energy2 unused when gridDim.y == 1).
__global__ void __launch_bounds__(128) k_energy(hdk_mesh m, hdk_material mat, const double* __restrict__ q1,
                                                 double* __restrict__ energy1, const double* __restrict__ q2,
                                                 double* __restrict__ energy2, int* bad) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const double* __restrict__ q = blockIdx.y ? q2 : q1;
  double* __restrict__ energy = blockIdx.y ? energy2 : energy1;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.ne) return;
  const ElemGeom g = load_geom(m, e);
  const M3 f = def_grad(g, q);
  // a segmented batch flags the element's own sample (hdk_ctl::bad of ctl[s],
  // sizeof(hdk_ctl) = 2 tau_stride ints apart)
  if (mat.seg_means) bad += (e / mat.seg_ne) * 2 * mat.tau_stride;
  if (!(det3(f) > 0.0)) {
    atomicCAS(bad, 0, 5);
    energy[e] = 0.0;
    return;
  }
  M3 u, v;
  V3 sf;
  signed_svd(f, u, sf, v);
  V3 s;
  if (!project(mat, e, sf, s)) {
    atomicCAS(bad, 0, 6);
    energy[e] = 0.0;
    return;
  }
  double dens;
  const V3 d = v3(s[0] - sf[0], s[1] - sf[1], s[2] - sf[2]);
  if (mat.kind == 1) {
    const Means mb = means_of(mat, e);
    const StretchNH den{mb.mu, mb.lambda};
    const double env = 0.5 * mb.k * dot3(d, d) + den.value(s);
    dens = mat.w1[e] / mb.k * env;  // w1 carries V
  } else {
    const V3 dev = v3(sf[0] - 1.0, sf[1] - 1.0, sf[2] - 1.0);
    dens = 0.5 * mat.w1[e] * dot3(dev, dev);  // mu_e V |sigma_F - 1|^2
    if (mat.barrier) {
      const double mu = mat.mu_e[e], la = mat.lambda_e[e], k = 2.0 * mu + la;
      const StretchBarrier den{mu, la};
      dens += mat.w2[e] / k * (0.5 * k * dot3(d, d) + den.value(s));
    } else {
      dens += 0.5 * mat.w2[e] * dot3(d, d);
    }
  }
  energy[e] = dens;
}

__device__ __forceinline__ void load_cache(const double* __restrict__ c, int ne, int e, V3& s, V3& sf, M3& u, M3& v) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    s[i] = c[(size_t)i * ne + e];
    sf[i] = c[(size_t)(3 + i) * ne + e];
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    u.m[i] = c[(size_t)(6 + i) * ne + e];
    v.m[i] = c[(size_t)(15 + i) * ne + e];
  }
}

// Compact differential D = {U, V, J (sym, 6), pair_a (3), pair_b (3)} with the
// element weight and volume folded into J and the pair coefficients.
__global__ void __launch_bounds__(128) k_differential(hdk_mesh m, hdk_material mat, const double* __restrict__ cache,
                                                       const double* tau_ptr, double* __restrict__ dcomp, int* err) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.ne) return;
  const int ne = m.ne;
  V3 s, sf;
  M3 u, v;
  load_cache(cache, ne, e, s, sf, u, v);
  M3 jac = m3_zero();
  double pa[3], pb[3];
  if (mat.kind == 1) {
    const Means mb = means_of(mat, e);
    const double tau = mat.seg_means ? tau_ptr[(e / mat.seg_ne) * mat.tau_stride] : *tau_ptr;
    const double k = mb.k, w = mat.w1[e];
    const StretchNH den{mb.mu, mb.lambda};
    M3 h = den.hessian(s);
    h(0, 0) += k; h(1, 1) += k; h(2, 2) += k;
    if (tau != 0.0) {  // tr_blend (localstep.cpp:286-303)
      V3 kap;
      M3 ev;
      sym_eig(h, kap, ev);
      V3 bl;
#pragma unroll
      for (int i = 0; i < 3; ++i) bl[i] = (1.0 - tau) * kap[i] + tau * fabs(kap[i]);
      h = eig_recompose(ev, bl);
    }
    V3 lam;
    M3 ev;
    sym_eig(h, lam, ev);  // nh_prox_differential (localstep.cpp:359-371)
    if (fmin(lam[0], fmin(lam[1], lam[2])) < 1e-12 * k) set_err(err, 7);
    jac = eig_recompose(ev, v3(w * k / lam[0], w * k / lam[1], w * k / lam[2]));
    pair_coefficients(sf, s, pa, pb);
#pragma unroll
    for (int i = 0; i < 3; ++i) { pa[i] *= w; pb[i] *= w; }
  } else {
    const double wr = mat.w1[e], wv = mat.w2[e];
    double ra[3], rb[3], va[3], vb[3];
    pair_coefficients(sf, v3(1.0, 1.0, 1.0), ra, rb);  // polar_differential
    pair_coefficients(sf, s, va, vb);
    if (mat.barrier) {  // barrier_differential (localstep.cpp:408-423)
      const double mu = mat.mu_e[e], la = mat.lambda_e[e], k = 2.0 * mu + la;
      const StretchBarrier den{mu, la};
      M3 h = den.hessian(s);
      h(0, 0) += k; h(1, 1) += k; h(2, 2) += k;
      V3 lam;
      M3 ev;
      sym_eig(h, lam, ev);
      if (fmin(lam[0], fmin(lam[1], lam[2])) < 1e-12 * k) set_err(err, 7);
      jac = eig_recompose(ev, v3(wv * k / lam[0], wv * k / lam[1], wv * k / lam[2]));
    } else {  // volume_differential (localstep.cpp:378-406)
      const V3 gr = v3(1.0 / s[0], 1.0 / s[1], 1.0 / s[2]);
      const double gamma = (gr[0] * (sf[0] - s[0]) + gr[1] * (sf[1] - s[1]) + gr[2] * (sf[2] - s[2])) / dot3(gr, gr);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double kkt[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) kkt[i] = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          kkt[i * 4 + i] = 1.0;
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (i != j) kkt[i * 4 + j] = gamma / (s[i] * s[j]);
          kkt[i * 4 + 3] = gr[i];
          kkt[12 + i] = gr[i];
        }
        double rhs[4] = {0.0, 0.0, 0.0, 0.0}, x[4];
        rhs[c] = 1.0;
        lu4_solve(kkt, rhs, x);
        jac(0, c) = x[0]; jac(1, c) = x[1]; jac(2, c) = x[2];
      }
      M3 sym;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) sym(r, c) = wv * 0.5 * (jac(r, c) + jac(c, r));
      jac = sym;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      pa[i] = wr * ra[i] + wv * va[i];
      pb[i] = wr * rb[i] + wv * vb[i];
    }
  }
  const size_t n = ne;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    dcomp[i * n + e] = u.m[i];
    dcomp[(9 + i) * n + e] = v.m[i];
  }
  dcomp[18 * n + e] = jac(0, 0);
  dcomp[19 * n + e] = jac(1, 1);
  dcomp[20 * n + e] = jac(2, 2);
  dcomp[21 * n + e] = 0.5 * (jac(0, 1) + jac(1, 0));
  dcomp[22 * n + e] = 0.5 * (jac(0, 2) + jac(2, 0));
  dcomp[23 * n + e] = 0.5 * (jac(1, 2) + jac(2, 1));
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    dcomp[(24 + i) * n + e] = pa[i];
    dcomp[(27 + i) * n + e] = pb[i];
  }
}

__device__ __forceinline__ M3 bforce(const ElemGeom& g, const double (&d)[30], const double* __restrict__ x);

// Element force of B x: P = U (D o (U^T F(x) V)) V^T, f_i = P g_i.
// Latency-bound (dependent index -> vertex gathers).  The block shape is a
// template for A/B runs (HETERODYN_BAPPLY): the unbounded 128-thread form
// (118 registers, more loads in flight per thread) measured faster at C3
// than register-capped single-wave shapes (10.0 vs 12.3 us per apply).
__device__ __forceinline__ void bapply_body(const hdk_mesh& m, const double* __restrict__ dcomp,
                                            const double* __restrict__ x, double* __restrict__ ef, const int* run_flag,
                                            const int* __restrict__ corner_pos) {
  // The element's geometry and differential do not depend on the previous
  // kernel (only x does): load them before the PDL wait, so they arrive
  // while that kernel drains.
  hdk::pdl_trigger();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = e < m.ne;
  const size_t n = m.ne;
  const int ee = live ? e : 0;
  const ElemGeom g = load_geom(m, ee);
  double d[30];
#pragma unroll
  for (int i = 0; i < 30; ++i) d[i] = __ldg(dcomp + i * n + ee);
  // the corners' slots are static too: no dependent load after the arithmetic
  const int4 pos = corner_pos ? __ldg(reinterpret_cast<const int4*>(corner_pos) + ee) : make_int4(0, 0, 0, 0);
  HDK_TRACED_WAIT(hdk::kTrBapply);
  if (run_flag && *run_flag == 0) return;
  if (!live) return;
  const M3 pm = bforce(g, d, x);
  if (corner_pos) write_force_at(g, pm, ef, pos);
  else write_force(g, pm, ef, e);
}

// The contact-adjoint columns' B p, all columns per thread: the element's
// geometry and differential are loaded once for the kColumns directions
// (column c at x + c x_stride, its sorted forces at ef + c ef_stride; a
// column whose CG has ended, cond0[c cond_stride] == 0, is skipped).
template <int K>
__global__ void __launch_bounds__(128) k_bapply_cols_fused(hdk_mesh m, const double* __restrict__ dcomp,
                                                           const double* __restrict__ x, size_t x_stride,
                                                           double* __restrict__ ef, size_t ef_stride,
                                                           const int* __restrict__ corner_pos, const int* cond0,
                                                           int cond_stride) {
  hdk::pdl_trigger();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = e < m.ne;
  const size_t n = m.ne;
  const int ee = live ? e : 0;
  const ElemGeom g = load_geom(m, ee);
  double d[30];
#pragma unroll
  for (int i = 0; i < 30; ++i) d[i] = __ldg(dcomp + i * n + ee);
  const int4 pos = __ldg(reinterpret_cast<const int4*>(corner_pos) + ee);
  hdk::pdl_wait();
  if (!live) return;
  const int c0 = K * blockIdx.y;  // column group of this block row
#pragma unroll 1
  for (int c = c0; c < c0 + K; ++c) {
    if (cond0[(size_t)c * cond_stride] == 0) continue;
    const M3 pm = bforce(g, d, x + c * x_stride);
    write_force_at(g, pm, ef + c * ef_stride, pos);
  }
}

// The element force of B x from the element's geometry and differential.
__device__ __forceinline__ M3 bforce(const ElemGeom& g, const double (&d)[30], const double* __restrict__ x) {
  const M3 df = def_grad(g, x);
  M3 u, v;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    u.m[i] = d[i];
    v.m[i] = d[9 + i];
  }
  const M3 hat = mul(mul_tn(u, df), v);
  const double j00 = d[18], j11 = d[19], j22 = d[20], j01 = d[21], j02 = d[22], j12 = d[23];
  M3 o;
  o(0, 0) = j00 * hat(0, 0) + j01 * hat(1, 1) + j02 * hat(2, 2);
  o(1, 1) = j01 * hat(0, 0) + j11 * hat(1, 1) + j12 * hat(2, 2);
  o(2, 2) = j02 * hat(0, 0) + j12 * hat(1, 1) + j22 * hat(2, 2);
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const int i = p == 2 ? 1 : 0, j = p == 0 ? 1 : 2;
    const double a = d[24 + p], b = d[27 + p];
    o(i, j) = a * hat(i, j) + b * hat(j, i);
    o(j, i) = b * hat(i, j) + a * hat(j, i);
  }
  return mul_nt(mul(u, o), v);
}

template <int T, int MINB>
__global__ void __launch_bounds__(T, MINB) k_bapply(hdk_mesh m, const double* __restrict__ dcomp, const double* __restrict__ x,
                                                 double* __restrict__ ef, const int* run_flag,
                                                 const int* __restrict__ corner_pos) {
  bapply_body(m, dcomp, x, ef, run_flag, corner_pos);
}

// B p of a segmented batch's CG: elements of samples whose CG has ended
// (cond0[sample cond_stride] == 0) write nothing.  The element data is
// loaded before the PDL wait as in bapply_body (issuing it after the flag
// read measured 159 vs 124 us per C5 apply: the prefetch overlap is worth
// more than the loads a finished sample saves).
__global__ void __launch_bounds__(128) k_bapply_seg(hdk_mesh m, const double* __restrict__ dcomp,
                                                    const double* __restrict__ x, double* __restrict__ ef,
                                                    const int* __restrict__ corner_pos, const int* cond0,
                                                    int cond_stride, int seg_ne) {
  hdk::pdl_trigger();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = e < m.ne;
  const size_t n = m.ne;
  const int ee = live ? e : 0;
  const ElemGeom g = load_geom(m, ee);
  double d[30];
#pragma unroll
  for (int i = 0; i < 30; ++i) d[i] = __ldg(dcomp + i * n + ee);
  const int4 pos = __ldg(reinterpret_cast<const int4*>(corner_pos) + ee);
  hdk::pdl_wait();
  if (!live) return;
  if (cond0[(size_t)(e / seg_ne) * cond_stride] == 0) return;
  const M3 pm = bforce(g, d, x);
  write_force_at(g, pm, ef, pos);
}

// B p of the contact-adjoint columns' CG (blockIdx.y = column): each column's
// direction by vertex at x + c x_stride, its sorted element forces at
// ef + c ef_stride; a column whose CG has ended (run flag at
// cond0[c cond_stride] == 0) does nothing.
__global__ void __launch_bounds__(128) k_bapply_cols_sorted(hdk_mesh m, const double* __restrict__ dcomp,
                                                            const double* __restrict__ x, size_t x_stride,
                                                            double* __restrict__ ef, size_t ef_stride,
                                                            const int* __restrict__ corner_pos, const int* cond0,
                                                            int cond_stride) {
  const int c = blockIdx.y;
  bapply_body(m, dcomp, x + c * x_stride, ef + c * ef_stride, cond0 + (size_t)c * cond_stride, corner_pos);
}

// B t of the contact-adjoint columns, blockIdx.y = column.
__global__ void __launch_bounds__(128) k_bapply_bbcols(hdk_mesh m, const double* __restrict__ dcomp, hdk_bb_columns c) {
  const hdk_bb_column& k = c.col[blockIdx.y];
  bapply_body(m, dcomp, k.tv, k.ef, &k.snap->cond, nullptr);
}

// Per-element gradient routing (backward.cpp:361-391) and the damping
// element force of mu (damping_rhs(mu), backward.cpp:311).
__global__ void __launch_bounds__(128) k_route_elem(hdk_mesh m, hdk_material mat, const double* __restrict__ cache,
                                                     const double* __restrict__ q_star, const double* __restrict__ mu,
                                                     double unit_mu, double unit_lambda, double* __restrict__ dl_dw,
                                                     double* __restrict__ dl_de, double* __restrict__ ef_damp) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.ne) return;
  const int ne = m.ne;
  const ElemGeom g = load_geom(m, e);
  const M3 gm = def_grad(g, mu);
  const M3 fs = def_grad(g, q_star);
  V3 s, sf;
  M3 u, v;
  load_cache(cache, ne, e, s, sf, u, v);
  const double vol = mat.vol[e];
  double against = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) against += gm.m[i] * fs.m[i];
  const M3 pstar = recompose(u, s, v);
  double dps = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) dps += gm.m[i] * pstar.m[i];
  if (mat.kind == 1) {
    const double w = vol * (dps - against);
    dl_dw[e] += w;
    dl_de[e] += (2.0 * unit_mu + unit_lambda) * w;
  } else {
    const M3 rot = mul_nt(u, v);
    double drot = 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) drot += gm.m[i] * rot.m[i];
    const double w1 = vol * (drot - against), w2 = vol * (dps - against);
    dl_dw[e] += w1;
    dl_dw[ne + e] += w2;
    dl_de[e] += 2.0 * unit_mu * w1 + unit_lambda * w2;
  }
  if (ef_damp) {
    const double c = mat.beta_vh ? mat.beta_vh[e] : 0.0;
    M3 p;
#pragma unroll
    for (int i = 0; i < 9; ++i) p.m[i] = c * gm.m[i];
    write_force(g, p, ef_damp, e);
  }
}

__global__ void __launch_bounds__(128) k_damp_elem(hdk_mesh m, const double* __restrict__ beta_vh,
                                                    const double* __restrict__ q, double* __restrict__ ef) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.ne) return;
  const ElemGeom g = load_geom(m, e);
  const M3 f = def_grad(g, q);
  const double c = beta_vh[e];
  M3 p;
#pragma unroll
  for (int i = 0; i < 9; ++i) p.m[i] = c * f.m[i];
  write_force(g, p, ef, e);
}

inline int blocks(int n, int t) { return (n + t - 1) / t; }

}  // namespace

extern "C" {

HDK_API int hdk_set_newton_eigen(int on) {
  return static_cast<int>(cudaMemcpyToSymbol(g_newton_eigen, &on, sizeof(int)));
}

HDK_API int hdk_local_step(const hdk_mesh* m, const hdk_material* mat, const double* q, double* elem_force,
                           double* cache, int* err, void* stream) {
  hdk::launch(k_local, dim3(blocks(m->ne, 128)), dim3(128), 0, static_cast<cudaStream_t>(stream), *m, *mat, q, elem_force, cache, err,
              static_cast<const hdk_ctl*>(nullptr), static_cast<const int*>(nullptr));
  return static_cast<int>(cudaGetLastError());
}
HDK_API int hdk_local_step_seg(const hdk_mesh* m, const hdk_material* mat, const double* q, double* elem_force,
                               int* err, const hdk_ctl* ctl, const int* corner_vpos, void* stream) {
  if (!mat->seg_means || mat->seg_ne <= 0 || !ctl) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_local, dim3(blocks(m->ne, 128)), dim3(128), 0, static_cast<cudaStream_t>(stream), *m, *mat, q, elem_force,
              static_cast<double*>(nullptr), err, ctl, corner_vpos);
  return static_cast<int>(cudaGetLastError());
}
HDK_API int hdk_local_step_sorted(const hdk_mesh* m, const hdk_material* mat, const double* q, double* elem_force,
                                  int* err, const int* corner_vpos, void* stream) {
  if (!corner_vpos) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_local, dim3(blocks(m->ne, 128)), dim3(128), 0, static_cast<cudaStream_t>(stream), *m, *mat, q, elem_force,
              static_cast<double*>(nullptr), err, static_cast<const hdk_ctl*>(nullptr), corner_vpos);
  return static_cast<int>(cudaGetLastError());
}

HDK_API int hdk_element_energy(const hdk_mesh* m, const hdk_material* mat, const double* q, double* energy, int* bad,
                               void* stream) {
  hdk::launch(k_energy, dim3(blocks(m->ne, 128)), dim3(128), 0, static_cast<cudaStream_t>(stream), *m, *mat, q, energy,
              q, energy, bad);
  return static_cast<int>(cudaGetLastError());
}

HDK_API int hdk_element_energy2(const hdk_mesh* m, const hdk_material* mat, const double* q1, double* energy1,
                                const double* q2, double* energy2, int* bad, void* stream) {
  hdk::launch(k_energy, dim3(blocks(m->ne, 128), 2), dim3(128), 0, static_cast<cudaStream_t>(stream), *m, *mat, q1,
              energy1, q2, energy2, bad);
  return static_cast<int>(cudaGetLastError());
}

HDK_API int hdk_differential(const hdk_mesh* m, const hdk_material* mat, const double* cache, const double* tau,
                             double* dcomp, int* err, void* stream) {
  hdk::launch(k_differential, dim3(blocks(m->ne, 128)), dim3(128), 0, static_cast<cudaStream_t>(stream), *m, *mat, cache, tau, dcomp, err);
  return static_cast<int>(cudaGetLastError());
}

HDK_API int hdk_bapply(const hdk_mesh* m, const double* dcomp, const double* x, double* elem_force, void* stream) {
  return hdk_bapply_flag(m, dcomp, x, elem_force, nullptr, stream);
}

HDK_API int hdk_bapply_flag(const hdk_mesh* m, const double* dcomp, const double* x, double* elem_force,
                            const int* run_flag, void* stream) {
  return hdk_bapply_sorted(m, dcomp, x, elem_force, nullptr, run_flag, stream);
}

HDK_API int hdk_bapply_cols_sorted(const hdk_mesh* m, const double* dcomp, const double* x, size_t x_stride,
                                   double* ef, size_t ef_stride, const int* corner_pos, const int* cond0,
                                   int cond_stride, int columns, void* stream) {
  static const bool fused = [] {
    const char* e = std::getenv("HETERODYN_BCOLS");  // "0": one column per blockIdx.y (A/B)
    return !(e && e[0] == '0');
  }();
  static const int per_thread = [] {  // columns per thread (HETERODYN_BCOLS_K: 8, 4 or 2)
    const char* e = std::getenv("HETERODYN_BCOLS_K");
    return e ? std::atoi(e) : 8;
  }();
  if (fused && columns == 8) {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (per_thread == 4)
      hdk::launch(k_bapply_cols_fused<4>, dim3(blocks(m->ne, 128), 2), dim3(128), 0, st, *m, dcomp, x, x_stride, ef,
                  ef_stride, corner_pos, cond0, cond_stride);
    else if (per_thread == 2)
      hdk::launch(k_bapply_cols_fused<2>, dim3(blocks(m->ne, 128), 4), dim3(128), 0, st, *m, dcomp, x, x_stride, ef,
                  ef_stride, corner_pos, cond0, cond_stride);
    else
      hdk::launch(k_bapply_cols_fused<8>, dim3(blocks(m->ne, 128)), dim3(128), 0, st, *m, dcomp, x, x_stride, ef,
                  ef_stride, corner_pos, cond0, cond_stride);
    return static_cast<int>(cudaGetLastError());
  }
  hdk::launch(k_bapply_cols_sorted, dim3(blocks(m->ne, 128), columns), dim3(128), 0, static_cast<cudaStream_t>(stream),
              *m, dcomp, x, x_stride, ef, ef_stride, corner_pos, cond0, cond_stride);
  return static_cast<int>(cudaGetLastError());
}

HDK_API int hdk_bapply_sorted_seg(const hdk_mesh* m, const double* dcomp, const double* x, double* elem_force,
                                  const int* corner_pos, const int* cond0, int cond_stride, int seg_ne, void* stream) {
  if (!corner_pos || !cond0 || seg_ne <= 0) return static_cast<int>(cudaErrorInvalidValue);
  hdk::launch(k_bapply_seg, dim3(blocks(m->ne, 128)), dim3(128), 0, static_cast<cudaStream_t>(stream), *m, dcomp, x,
              elem_force, corner_pos, cond0, cond_stride, seg_ne);
  return static_cast<int>(cudaGetLastError());
}
HDK_API int hdk_bapply_sorted(const hdk_mesh* m, const double* dcomp, const double* x, double* elem_force,
                              const int* corner_pos, const int* run_flag, void* stream) {
  static const int variant = [] {
    const char* v = std::getenv("HETERODYN_BAPPLY");
    return v ? std::atoi(v) : 0;
  }();
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (variant == 0)
    hdk::launch(k_bapply<128, 1>, dim3(blocks(m->ne, 128)), dim3(128), 0, st, *m, dcomp, x, elem_force, run_flag, corner_pos);
  else if (variant == 2)
    hdk::launch(k_bapply<128, 6>, dim3(blocks(m->ne, 128)), dim3(128), 0, st, *m, dcomp, x, elem_force, run_flag, corner_pos);
  else
    hdk::launch(k_bapply<64, 11>, dim3(blocks(m->ne, 64)), dim3(64), 0, st, *m, dcomp, x, elem_force, run_flag, corner_pos);
  return static_cast<int>(cudaGetLastError());
}

HDK_API int hdk_bb_columns_bapply(const hdk_mesh* m, const double* dcomp, const hdk_bb_columns* c, void* stream) {
  hdk::launch(k_bapply_bbcols, dim3(blocks(m->ne, 128), HDK_BB_COLUMNS), dim3(128), 0,
              static_cast<cudaStream_t>(stream), *m, dcomp, *c);
  return static_cast<int>(cudaGetLastError());
}

HDK_API int hdk_route_elements(const hdk_mesh* m, const hdk_material* mat, const double* cache, const double* q_star,
                               const double* mu, double unit_mu, double unit_lambda, double* dl_dw, double* dl_de,
                               double* ef_damp, void* stream) {
  hdk::launch(k_route_elem, dim3(blocks(m->ne, 128)), dim3(128), 0, static_cast<cudaStream_t>(stream), *m, *mat, cache, q_star, mu, unit_mu, unit_lambda, dl_dw, dl_de, ef_damp);
  return static_cast<int>(cudaGetLastError());
}

HDK_API int hdk_damping_elements(const hdk_mesh* m, const double* beta_vh, const double* q, double* elem_force,
                                 void* stream) {
  hdk::launch(k_damp_elem, dim3(blocks(m->ne, 128)), dim3(128), 0, static_cast<cudaStream_t>(stream), *m, beta_vh, q, elem_force);
  return static_cast<int>(cudaGetLastError());
}

}  // extern "C"
