// Contact kernels (reference contact.cpp, forward.cpp:171-235,
// backward.cpp:227-283): vertex-vs-analytic-obstacle detection, Fischer-
// Burmeister NCP weights, the lifted multiplier system, block cone
// projection, and the contact-corrected iterate.  Rows follow the
// reference's stacked order: normals, bilateral (none from detection), then
// two tangent rows per frictional contact.  The dense K x K factorization is
// a Cholesky (the system is SPD; the reference's pivoted LDLT agrees to
// rounding) done by cuSOLVER from the host engine.
#include <cuda_runtime.h>

#include <cmath>

#include "../../include/hdk.h"
#include "launch.cuh"

namespace {

constexpr int kT = 256;

// Signed distance of every (free vertex, obstacle) pair at q; flags[v*no+o] = 1
// when sd <= margin (contact.cpp:126-133).
__global__ void k_detect(int nv, const int* v2p, const double* q, int no, const double* obs, double margin,
                         unsigned char* flags) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv * no) return;
  const int v = i / no, o = i - v * no;
  if (v2p[v] < 0) {
    flags[i] = 0;
    return;
  }
  const double* ob = obs + 8 * o;  // kind, nx, ny, nz, offset|radius, cx, cy, cz
  const double x = q[3 * v], y = q[3 * v + 1], z = q[3 * v + 2];
  double sd;
  if (ob[0] == 0.0) {
    sd = ob[1] * x + ob[2] * y + ob[3] * z - ob[4];
  } else {
    const double dx = x - ob[5], dy = y - ob[6], dz = z - ob[7];
    sd = sqrt(dx * dx + dy * dy + dz * dz) - ob[4];
  }
  flags[i] = sd <= margin ? 1 : 0;
}

__device__ __forceinline__ void ncp(double delta, double r, double lambda, double& om, double& e) {
  const double root = sqrt(delta * delta + r * r * lambda * lambda);
  if (root == 0.0) {  // active-branch limit at the origin (contact.cpp:154)
    om = 1.0;
    e = r;
    return;
  }
  om = 1.0 - delta / root;
  e = (1.0 - r * lambda / root) * r;
}

// NCP weights per row (contact_weights, contact.cpp:160-196).
__global__ void k_weights(hdk_contacts c, const double* q, const double* qt, const double* lambda, double* omega,
                          double* e_diag) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < c.nc) {
    const int v = c.vertex[i];
    const double* n = c.normal + 3 * i;
    const double delta = n[0] * q[3 * v] + n[1] * q[3 * v + 1] + n[2] * q[3 * v + 2] - c.gap[i];
    double om, e;
    ncp(delta, c.r_n[i], lambda[i], om, e);
    omega[i] = om;
    e_diag[i] = e;
  }
  if (i < c.nf) {
    const int ci = c.fric[i];
    const int v = c.vertex[ci];
    const double* t1 = c.t1 + 3 * ci;
    const double* t2 = c.t2 + 3 * ci;
    const double d0 = q[3 * v] - qt[3 * v], d1 = q[3 * v + 1] - qt[3 * v + 1], d2 = q[3 * v + 2] - qt[3 * v + 2];
    const double slip = hypot(t1[0] * d0 + t1[1] * d1 + t1[2] * d2, t2[0] * d0 + t2[1] * d1 + t2[2] * d2);
    const int row = c.nc + 2 * i;
    const double lam_n = lambda[ci];
    const double lam_f = hypot(lambda[row], lambda[row + 1]);
    const double slack = c.mu[ci] * lam_n - lam_f;
    double om, e;
    ncp(slip, c.r_f[ci], slack, om, e);
    omega[row] = omega[row + 1] = om;
    e_diag[row] = e_diag[row + 1] = e;
  }
}

// Row directions and vertices of the stacked rows.
__device__ __forceinline__ void row_of(const hdk_contacts& c, int r, int& v, const double*& d) {
  if (r < c.nc) {
    v = c.vertex[r];
    d = c.normal + 3 * r;
  } else {
    const int f = (r - c.nc) >> 1;
    const int ci = c.fric[f];
    v = c.vertex[ci];
    d = ((r - c.nc) & 1) ? c.t2 + 3 * ci : c.t1 + 3 * ci;
  }
}

// jq[r] = d_r . q[v_r]  (ContactSet::constraint_values, contact.cpp:100-115)
__global__ void k_jq(hdk_contacts c, const double* q, double* jq) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= c.k) return;
  int v;
  const double* d;
  row_of(c, r, v, d);
  jq[r] = d[0] * q[3 * v] + d[1] * q[3 * v + 1] + d[2] * q[3 * v + 2];
}

// System of one multiplier update (contact_iteration, contact.cpp:237-256):
// M = Omega W Omega + diag(E) + lift I (column-major, lower used),
// rhs = h_vec - omega o (J q0 + W (omega o lambda)) with
// h_vec = offset_vector (contact.cpp:198-216).  J q_mid is formed exactly as
// J q0 + W (omega o lambda) since the correction is A^{-1} J^T (omega o lambda).
__global__ void __launch_bounds__(kT) k_system(hdk_contacts c, const double* W, const double* omega,
                                               const double* e_diag, const double* lambda, const double* jq0,
                                               const double* qt, double* M, double* rhs) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int k = c.k;
  __shared__ double red[kT / 32];
  __shared__ double lift_sh;
  // trace of Omega W Omega + E (fixed-order block reduction)
  double t = 0.0;
  for (int r = threadIdx.x; r < k; r += kT) t += omega[r] * W[(size_t)r * k + r] * omega[r] + e_diag[r];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kT / 32; ++w) s += red[w];
    lift_sh = 1e-10 * s / k;
  }
  __syncthreads();
  const double lift = lift_sh;
  for (size_t idx = threadIdx.x; idx < (size_t)k * k; idx += kT) {
    const int col = static_cast<int>(idx / k), row = static_cast<int>(idx % k);
    double m = omega[row] * W[idx] * omega[col];
    if (row == col) m += e_diag[row] + lift;
    M[idx] = m;
  }
  for (int r = threadIdx.x; r < k; r += kT) {
    double wl = 0.0;
    for (int s = 0; s < k; ++s) wl += W[(size_t)s * k + r] * (omega[s] * lambda[s]);
    double h;
    if (r < c.nc) {
      h = omega[r] * c.gap[r];
    } else {
      int v;
      const double* d;
      row_of(c, r, v, d);
      h = omega[r] * (d[0] * qt[3 * v] + d[1] * qt[3 * v + 1] + d[2] * qt[3 * v + 2]);
    }
    rhs[r] = h - omega[r] * (jq0[r] + wl);
  }
}

// lambda <- project(lambda + step): normals clamped, friction pairs radially
// scaled into mu * lambda_n (project_multipliers, contact.cpp:218-235).
__global__ void k_project(hdk_contacts c, const double* step, double* lambda, int* err) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < c.k; r += blockDim.x) {
    const double nl = lambda[r] + step[r];
    if (!isfinite(step[r])) bad = 1;
    lambda[r] = nl;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < c.nc; i += blockDim.x) lambda[i] = fmax(0.0, lambda[i]);
  __syncthreads();
  for (int f = threadIdx.x; f < c.nf; f += blockDim.x) {
    const int ci = c.fric[f];
    const int row = c.nc + 2 * f;
    const double bound = c.mu[ci] * lambda[ci];
    const double lf = hypot(lambda[row], lambda[row + 1]);
    if (lf > bound) {
      const double sc = bound > 0 ? bound / lf : 0.0;
      lambda[row] *= sc;
      lambda[row + 1] *= sc;
    }
  }
  if (threadIdx.x == 0 && bad && err) atomicCAS(err, 0, 9);
}

// g_u = sum over rows r at unique vertex u of coef_r d_r, coef = omega o lambda.
__global__ void k_vertex_coef(hdk_contacts c, const double* omega, const double* lambda, double scale, double* g) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= c.nu) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int j = c.urow_off[u]; j < c.urow_off[u + 1]; ++j) {
    const int r = c.urow[j];
    int v;
    const double* d;
    row_of(c, r, v, d);
    const double coef = scale * omega[r] * lambda[r];
    s0 += coef * d[0];
    s1 += coef * d[1];
    s2 += coef * d[2];
  }
  g[3 * u] = s0;
  g[3 * u + 1] = s1;
  g[3 * u + 2] = s2;
}

// out[v] = base[v] + sum_u U[p(v), u] g_u on free vertices (contact_corrected,
// forward.cpp:196-206, through the cached scalar columns U = A_s^{-1} E).
__global__ void k_corrected(int n, const int* p2v, const double* U, int nu, const double* g, const double* base,
                            double* out) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int u = 0; u < nu; ++u) {
    const double w = U[(size_t)u * n + p];
    s0 += w * g[3 * u];
    s1 += w * g[3 * u + 1];
    s2 += w * g[3 * u + 2];
  }
  const int v = p2v[p];
  out[3 * v] = base[3 * v] + s0;
  out[3 * v + 1] = base[3 * v + 1] + s1;
  out[3 * v + 2] = base[3 * v + 2] + s2;
}

// Scalar inverse columns: U[:, u] = A_s^{-1} e_{p(u)}; scatter unit spikes of
// three vertices at a time into the three axes of one solve right-hand side.
__global__ void k_spikes(int n, const int* up, int u0, int cnt, double* rhs_perm) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  for (int a = 0; a < 3; ++a) rhs_perm[3 * (size_t)p + a] = (a < cnt && up[u0 + a] == p) ? 1.0 : 0.0;
}
__global__ void k_unspike(int n, const double* x_perm, int u0, int cnt, double* U) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  for (int a = 0; a < cnt; ++a) U[(size_t)(u0 + a) * n + p] = x_perm[3 * (size_t)p + a];
}

// W(r, s) = (d_r . d_s) U[p(u_s), u_r] (Delassus, factor.cpp:237-289).
__global__ void k_delassus(hdk_contacts c, const double* U, int n, const int* up, double* W) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (idx >= (size_t)c.k * c.k) return;
  const int s = static_cast<int>(idx / c.k), r = static_cast<int>(idx % c.k);
  int vr, vs;
  const double *dr, *ds;
  row_of(c, r, vr, dr);
  row_of(c, s, vs, ds);
  const int ur = c.row_unique[r], us = c.row_unique[s];
  const int ua = ur < us ? ur : us, ub = ur < us ? us : ur;  // one triangle, mirrored (factor.cpp:283-285)
  W[idx] = (dr[0] * ds[0] + dr[1] * ds[1] + dr[2] * ds[2]) * U[(size_t)ua * n + up[ub]];
}

// Adjoint contact elimination (backward.cpp:240-283): w_tan(d, c) = d_d . X_c[v_d],
// symmetrised; M = Omega sym Omega + diag(E) + lift I; rhs = omega o (J z0).
__global__ void __launch_bounds__(kT) k_reduced(hdk_contacts c, const double* X, size_t ldx, const double* omega,
                                                const double* e_diag, const double* z0, double* M, double* rhs) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int k = c.k;
  __shared__ double red[kT / 32];
  __shared__ double lift_sh;
  auto wt = [&](int d, int col) {
    int v;
    const double* dir;
    row_of(c, d, v, dir);
    const double* x = X + (size_t)col * ldx + 3 * (size_t)v;
    return dir[0] * x[0] + dir[1] * x[1] + dir[2] * x[2];
  };
  double t = 0.0;
  for (int r = threadIdx.x; r < k; r += kT) t += omega[r] * wt(r, r) * omega[r] + e_diag[r];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kT / 32; ++w) s += red[w];
    lift_sh = 1e-10 * s / k;
  }
  __syncthreads();
  for (size_t idx = threadIdx.x; idx < (size_t)k * k; idx += kT) {
    const int col = static_cast<int>(idx / k), row = static_cast<int>(idx % k);
    const double sym = 0.5 * (wt(row, col) + wt(col, row));
    double m = omega[row] * sym * omega[col];
    if (row == col) m += e_diag[row] + lift_sh;
    M[idx] = m;
  }
  for (int r = threadIdx.x; r < k; r += kT) {
    int v;
    const double* d;
    row_of(c, r, v, d);
    rhs[r] = omega[r] * (d[0] * z0[3 * v] + d[1] * z0[3 * v + 1] + d[2] * z0[3 * v + 2]);
  }
}

// mu = z0 - sum_c (omega_c y_c) X_c (backward.cpp:266-268); nonfinite y -> error.
__global__ void k_combine(int n3, const double* z0, const double* X, size_t ldx, int k, const double* omega,
                          const double* y, double* mu, int* err) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  double s = z0[i];
  for (int c = 0; c < k; ++c) s -= (omega[c] * y[c]) * X[(size_t)c * ldx + i];
  mu[i] = s;
  if (i == 0) {
    for (int c = 0; c < k; ++c)
      if (!isfinite(y[c])) {
        atomicCAS(err, 0, 10);
        break;
      }
  }
}

// Column right-hand side and warm start of row c: rhs = e_v d_c (full),
// x0 = a_c = U[:, slot] d_c on free vertices, zero on fixed ones.
__global__ void k_column_init(hdk_contacts c, int row, int nv, const int* v2p, const double* U, int n, double* rhs,
                              double* x0) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  int vr;
  const double* d;
  row_of(c, row, vr, d);
  const int p = v2p[v];
  const double u = p >= 0 ? U[(size_t)c.row_unique[row] * n + p] : 0.0;
  for (int a = 0; a < 3; ++a) {
    rhs[3 * v + a] = v == vr ? d[a] : 0.0;
    x0[3 * v + a] = u * d[a];
  }
}

// Friction rows push back into q_t (backward.cpp:342-356).
__global__ void k_friction_pushback(hdk_contacts c, const double* omega, const double* y, double* dl_dq) {
  hdk::pdl_wait();
  hdk::pdl_trigger();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int f = 0; f < c.nf; ++f)
    for (int t = 0; t < 2; ++t) {
      const int row = c.nc + 2 * f + t;
      int v;
      const double* d;
      row_of(c, row, v, d);
      const double w = omega[row] * y[row];
      dl_dq[3 * v] += w * d[0];
      dl_dq[3 * v + 1] += w * d[1];
      dl_dq[3 * v + 2] += w * d[2];
    }
}

inline int nb(long long n) { return static_cast<int>((n + 255) / 256); }
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
inline int last() { return static_cast<int>(cudaGetLastError()); }

}  // namespace

extern "C" {

HDK_API int hdk_contact_detect(int nv, const int* v2p, const double* q, int n_obstacles, const double* obstacles,
                               double margin, unsigned char* flags, void* stream) {
  if (nv * n_obstacles == 0) return 0;
  hdk::launch(k_detect, dim3(nb(static_cast<long long>(nv) * n_obstacles)), dim3(256), 0, S(stream), nv, v2p, q,
              n_obstacles, obstacles, margin, flags);
  return last();
}

HDK_API int hdk_contact_weights(const hdk_contacts* c, const double* q, const double* q_t, const double* lambda,
                                double* omega, double* e_diag, void* stream) {
  hdk::launch(k_weights, dim3(nb(c->nc > c->nf ? c->nc : c->nf)), dim3(256), 0, S(stream), *c, q, q_t, lambda, omega,
              e_diag);
  return last();
}

HDK_API int hdk_contact_jq(const hdk_contacts* c, const double* q, double* jq, void* stream) {
  hdk::launch(k_jq, dim3(nb(c->k)), dim3(256), 0, S(stream), *c, q, jq);
  return last();
}

HDK_API int hdk_contact_system(const hdk_contacts* c, const double* W, const double* omega, const double* e_diag,
                               const double* lambda, const double* jq0, const double* q_t, double* M, double* rhs,
                               void* stream) {
  hdk::launch(k_system, dim3(1), dim3(kT), 0, S(stream), *c, W, omega, e_diag, lambda, jq0, q_t, M, rhs);
  return last();
}

HDK_API int hdk_contact_project(const hdk_contacts* c, const double* step, double* lambda, int* err, void* stream) {
  hdk::launch(k_project, dim3(1), dim3(256), 0, S(stream), *c, step, lambda, err);
  return last();
}

HDK_API int hdk_contact_correct(const hdk_contacts* c, int n, const int* p2v, const double* U, const double* omega,
                                const double* lambda, double scale, double* g, const double* base, double* out,
                                void* stream) {
  hdk::launch(k_vertex_coef, dim3(nb(c->nu)), dim3(256), 0, S(stream), *c, omega, lambda, scale, g);
  hdk::launch(k_corrected, dim3(nb(n)), dim3(256), 0, S(stream), n, p2v, U, c->nu, static_cast<const double*>(g), base,
              out);
  return last();
}

HDK_API int hdk_contact_spikes(int n, const int* unique_pos, int u0, int count, double* rhs_perm, void* stream) {
  hdk::launch(k_spikes, dim3(nb(n)), dim3(256), 0, S(stream), n, unique_pos, u0, count, rhs_perm);
  return last();
}

HDK_API int hdk_contact_unspike(int n, const double* x_perm, int u0, int count, double* U, void* stream) {
  hdk::launch(k_unspike, dim3(nb(n)), dim3(256), 0, S(stream), n, x_perm, u0, count, U);
  return last();
}

HDK_API int hdk_contact_delassus(const hdk_contacts* c, const double* U, int n, const int* unique_pos, double* W,
                                 void* stream) {
  hdk::launch(k_delassus, dim3(nb(static_cast<long long>(c->k) * c->k)), dim3(256), 0, S(stream), *c, U, n, unique_pos,
              W);
  return last();
}

HDK_API int hdk_contact_reduced(const hdk_contacts* c, const double* X, size_t ldx, const double* omega,
                                const double* e_diag, const double* z0, double* M, double* rhs, void* stream) {
  hdk::launch(k_reduced, dim3(1), dim3(kT), 0, S(stream), *c, X, ldx, omega, e_diag, z0, M, rhs);
  return last();
}

HDK_API int hdk_contact_combine(int n3, const double* z0, const double* X, size_t ldx, int k, const double* omega,
                                const double* y, double* mu, int* err, void* stream) {
  hdk::launch(k_combine, dim3(nb(n3)), dim3(256), 0, S(stream), n3, z0, X, ldx, k, omega, y, mu, err);
  return last();
}

HDK_API int hdk_contact_column_init(const hdk_contacts* c, int row, int nv, const int* v2p, const double* U, int n,
                                    double* rhs, double* x0, void* stream) {
  hdk::launch(k_column_init, dim3(nb(nv)), dim3(256), 0, S(stream), *c, row, nv, v2p, U, n, rhs, x0);
  return last();
}

HDK_API int hdk_contact_friction_pushback(const hdk_contacts* c, const double* omega, const double* y, double* dl_dq,
                                          void* stream) {
  hdk::launch(k_friction_pushback, dim3(1), dim3(32), 0, S(stream), *c, omega, y, dl_dq);
  return last();
}

}  // extern "C"
