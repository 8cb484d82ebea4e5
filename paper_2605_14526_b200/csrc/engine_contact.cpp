// Contact path of the device engine and the per-frame adjoint driver.
//
// Forward (forward.cpp:171-235): detection at the free-fall target on the
// device (flags) in the reference's vertex-major / obstacle-minor order; the
// contact geometry (normal, gap offset, tangent basis — contact.cpp:46-66,
// 117-144) is assembled on the host from the flagged rows; the scalar inverse
// columns of the contact vertices come from the same explicit-factor solve,
// three unit spikes per 3-axis application; the Delassus matrix and the
// per-iteration multiplier update run on the device (dense Cholesky through
// cuSOLVER for the lifted K x K system).
//
// Backward (backward.cpp:208-284): the backbone adjoint z0, one warm-started
// backbone per contact row, the reduced multiplier system and the friction
// pushback, all on the device through the same graphs as the contact-free
// path.
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "engine.hpp"

namespace hdb {

namespace {
void hdk_check(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }
void sol_check(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS) raise(Code::InvalidArgument, std::string("cuSOLVER failure in ") + what);
}
inline P3 sub(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double dot(P3 a, P3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline P3 cross(P3 a, P3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double norm(P3 a) { return std::sqrt(dot(a, a)); }

// Signed distance and outward normal of an obstacle (contact.cpp:39-52).
double signed_distance(const Obstacle& o, P3 x) {
  if (o.kind == 0) return dot(o.normal, x) - o.offset;
  return norm(sub(x, o.center)) - o.radius;
}
P3 outward_normal(const Obstacle& o, P3 x) {
  if (o.kind == 0) return o.normal;
  const P3 d = sub(x, o.center);
  const double len = norm(d);
  if (len < 1e-12) return {0, 1, 0};
  return {d.x / len, d.y / len, d.z / len};
}
// Deterministic tangent basis (contact.cpp:54-66).
void tangents(P3 n, P3& t1, P3& t2) {
  const P3 a{std::fabs(n.x), std::fabs(n.y), std::fabs(n.z)};
  P3 axis{1, 0, 0};
  if (a.y <= a.x && a.y <= a.z) axis = {0, 1, 0};
  else if (a.z <= a.x && a.z <= a.y) axis = {0, 0, 1};
  t1 = cross(n, axis);
  const double l = norm(t1);
  t1 = {t1.x / l, t1.y / l, t1.z / l};
  t2 = cross(n, t1);
}
}  // namespace

void Engine::ensure_solver_workspace(int k) {
  if (!cusolver_) {
    cusolverDnHandle_t hnd;
    sol_check(cusolverDnCreate(&hnd), "create");
    cusolver_ = hnd;
    cuda_check(cudaMalloc(&cinfo_, sizeof(int)), "cusolver info");
  }
  auto hnd = static_cast<cusolverDnHandle_t>(cusolver_);
  sol_check(cusolverDnSetStream(hnd, st_), "set stream");
  if (k <= c_cap_) return;
  const int cap = std::max(k, 2 * c_cap_);
  for (double** p : {&cjq_, &cM_, &crhs_, &cg_})
    if (*p) cudaFree(*p);
  cuda_check(cudaMalloc(&cjq_, sizeof(double) * cap), "contact buffers");
  cuda_check(cudaMalloc(&cM_, sizeof(double) * static_cast<size_t>(cap) * cap), "contact buffers");
  cuda_check(cudaMalloc(&crhs_, sizeof(double) * cap), "contact buffers");
  cuda_check(cudaMalloc(&cg_, sizeof(double) * 3 * cap), "contact buffers");
  int lwork = 0;
  sol_check(cusolverDnDpotrf_bufferSize(hnd, CUBLAS_FILL_MODE_LOWER, cap, cM_, cap, &lwork), "potrf buffer");
  if (lwork > cwork_len_) {
    if (cwork_) cudaFree(cwork_);
    cuda_check(cudaMalloc(&cwork_, sizeof(double) * std::max(lwork, 1)), "cusolver work");
    cwork_len_ = lwork;
  }
  c_cap_ = cap;
}

std::shared_ptr<ContactFrame> Engine::detect_and_setup() {
  const int nv = scene_.mesh.nv, no = static_cast<int>(scene_.obstacles.size());
  const size_t n3 = 3 * static_cast<size_t>(nv);
  hdk_check(hdk_contact_detect(nv, df_.v2p, qtil_, no, obst_, scene_.solver.contact_margin, flags_, st_), "detect");
  std::vector<unsigned char> flags(static_cast<size_t>(nv) * no);
  Vec qt(n3);
  cuda_check(cudaMemcpyAsync(flags.data(), flags_, flags.size(), cudaMemcpyDeviceToHost, st_), "flags");
  cuda_check(cudaMemcpyAsync(qt.data(), qtil_, n3 * sizeof(double), cudaMemcpyDeviceToHost, st_), "q tilde");
  cuda_check(cudaStreamSynchronize(st_), "detect sync");
  auto cf = std::make_shared<ContactFrame>();
  ContactFrame& c = *cf;
  for (int v = 0; v < nv; ++v)
    for (int o = 0; o < no; ++o) {
      if (!flags[static_cast<size_t>(v) * no + o]) continue;
      const Obstacle& ob = scene_.obstacles[o];
      const P3 x{qt[3 * v], qt[3 * v + 1], qt[3 * v + 2]};
      const P3 nrm = outward_normal(ob, x);
      P3 t1, t2;
      tangents(nrm, t1, t2);
      c.vertex.push_back(v);
      for (double d : {nrm.x, nrm.y, nrm.z}) c.normal.push_back(d);
      for (double d : {t1.x, t1.y, t1.z}) c.t1.push_back(d);
      for (double d : {t2.x, t2.y, t2.z}) c.t2.push_back(d);
      c.gap.push_back(dot(nrm, x) - signed_distance(ob, x));
      c.mu.push_back(ob.friction);
    }
  c.nc = static_cast<int>(c.vertex.size());
  for (int i = 0; i < c.nc; ++i)
    if (c.mu[i] > 0) c.fric.push_back(i);
  c.nf = static_cast<int>(c.fric.size());
  c.k = c.nc + 2 * c.nf;
  if (c.k == 0) return cf;
  // unique vertices in order of first appearance over the stacked rows
  std::vector<int> slot(nv, -1);
  c.row_unique.resize(c.k);
  auto row_vertex = [&](int r) { return r < c.nc ? c.vertex[r] : c.vertex[c.fric[(r - c.nc) >> 1]]; };
  for (int r = 0; r < c.k; ++r) {
    const int v = row_vertex(r);
    if (slot[v] < 0) {
      slot[v] = static_cast<int>(c.unique_vertex.size());
      c.unique_vertex.push_back(v);
      c.unique_pos.push_back(hf_.v2p[v]);
    }
    c.row_unique[r] = slot[v];
  }
  c.nu = static_cast<int>(c.unique_vertex.size());
  c.urow_off.assign(c.nu + 1, 0);
  for (int r = 0; r < c.k; ++r) ++c.urow_off[c.row_unique[r] + 1];
  for (int u = 0; u < c.nu; ++u) c.urow_off[u + 1] += c.urow_off[u];
  c.urow.resize(c.k);
  {
    std::vector<int> cur(c.urow_off.begin(), c.urow_off.end() - 1);
    for (int r = 0; r < c.k; ++r) c.urow[cur[c.row_unique[r]]++] = r;
  }
  c.r_n.assign(c.nc, 0.0);
  c.r_f.assign(c.nc, 0.0);
  // device view (r_n / r_f filled after the Delassus matrix)
  c.mem = std::make_unique<DevArena>();
  DevArena& A = *c.mem;
  const int n = hf_.n;
  c.view.nc = c.nc;
  c.view.nf = c.nf;
  c.view.k = c.k;
  c.view.nu = c.nu;
  c.view.vertex = A.upload(c.vertex);
  c.view.normal = A.upload(c.normal);
  c.view.t1 = A.upload(c.t1);
  c.view.t2 = A.upload(c.t2);
  c.view.gap = A.upload(c.gap);
  c.view.mu = A.upload(c.mu);
  double* rn = A.alloc<double>(c.nc);
  double* rf = A.alloc<double>(c.nc);
  c.view.r_n = rn;
  c.view.r_f = rf;
  c.view.fric = A.upload(c.fric.empty() ? std::vector<int>{0} : c.fric);
  c.view.row_unique = A.upload(c.row_unique);
  c.view.urow_off = A.upload(c.urow_off);
  c.view.urow = A.upload(c.urow);
  c.unique_pos_d = A.upload(c.unique_pos);
  c.U = A.alloc<double>(static_cast<size_t>(n) * c.nu);
  c.W = A.alloc<double>(static_cast<size_t>(c.k) * c.k);
  c.lambda = A.alloc<double>(c.k);
  c.omega = A.alloc<double>(c.k);
  c.e_diag = A.alloc<double>(c.k);
  // scalar inverse columns: three unit spikes per 3-axis solve
  for (int u0 = 0; u0 < c.nu; u0 += 3) {
    const int cnt = std::min(3, c.nu - u0);
    hdk_check(hdk_contact_spikes(n, c.unique_pos_d, u0, cnt, rhs_, st_), "spikes");
    hdk_check(hdk_apply_inverse3_perm(&df_, rhs_, dqp_, st_), "inverse columns");
    hdk_check(hdk_contact_unspike(n, dqp_, u0, cnt, c.U, st_), "unspike");
    ++solve_count;
    kernel_launches += 6;
  }
  hdk_check(hdk_contact_delassus(&c.view, c.U, n, c.unique_pos_d, c.W, st_), "delassus");
  ++kernel_launches;
  // r_n = h^2 W_nn, r_f = h^2 (W_tt1 + W_tt2)/2 (forward.cpp:183-192)
  Vec diag(c.k);
  cuda_check(cudaMemcpy2DAsync(diag.data(), sizeof(double), c.W, sizeof(double) * (c.k + 1), sizeof(double), c.k,
                               cudaMemcpyDeviceToHost, st_), "W diagonal");
  cuda_check(cudaStreamSynchronize(st_), "W diagonal");
  const double h = scene_.solver.h;
  for (int i = 0; i < c.nc; ++i) c.r_n[i] = h * h * diag[i];
  for (int f = 0; f < c.nf; ++f) {
    const int fr = c.nc + 2 * f;
    c.r_f[c.fric[f]] = h * h * 0.5 * (diag[fr] + diag[fr + 1]);
  }
  DevArena::copy_h2d(rn, c.r_n.data(), sizeof(double) * c.nc);
  DevArena::copy_h2d(rf, c.r_f.data(), sizeof(double) * c.nc);
  return cf;
}

// PD loop with the contact update inside (forward.cpp:222-250), launched
// kernel by kernel with one status read per iteration.
void Engine::contact_loop(ContactFrame& c) {
  const Solver& so = scene_.solver;
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  const double h = so.h;
  const int n = hf_.n, k = c.k;
  ensure_solver_workspace(k);
  auto hnd = static_cast<cusolverDnHandle_t>(cusolver_);
  void* s = st_;
  cuda_check(cudaMemsetAsync(c.lambda, 0, sizeof(double) * k, st_), "lambda zero");
  cuda_check(cudaMemcpyAsync(q0c_, q_, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st_), "q0 init");
  hdk_check(hdk_ctl_init(ctl_, aa_window_, 10.0, so.k_max, so.eps_rel, so.eps_abs, 0.0, so.eps_tr, 0, s), "ctl init");
  int host_info = 0;
  for (int it = 0; it < so.k_max; ++it) {
    hdk_check(hdk_local_step(&dm_, &dmat_, qcur_, ef_, nullptr, &ctl_->err, s), "local step");
    hdk_check(hdk_gather_rhs(&dv_, ef_, 1.0 / (h * h), qtil_, damp_, hf_.fixed.empty() ? nullptr : fixc_, bprev_, rhs_,
                             part_a_, s), "rhs");
    hdk_check(hdk_apply_inverse3(&df_, rhs_, q0c_, s), "solve");
    hdk_check(hdk_contact_weights(&c.view, qcur_, q_, c.lambda, c.omega, c.e_diag, s), "weights");
    hdk_check(hdk_contact_jq(&c.view, q0c_, cjq_, s), "J q0");
    hdk_check(hdk_contact_system(&c.view, c.W, c.omega, c.e_diag, c.lambda, cjq_, q_, cM_, crhs_, s), "system");
    sol_check(cusolverDnDpotrf(hnd, CUBLAS_FILL_MODE_LOWER, k, cM_, k, cwork_, cwork_len_, cinfo_), "potrf");
    sol_check(cusolverDnDpotrs(hnd, CUBLAS_FILL_MODE_LOWER, k, 1, cM_, k, crhs_, k, cinfo_), "potrs");
    hdk_check(hdk_contact_project(&c.view, crhs_, c.lambda, &ctl_->err, s), "project");
    hdk_check(hdk_contact_correct(&c.view, n, df_.p2v, c.U, c.omega, c.lambda, 1.0, cg_, q0c_, qhat_, s), "q hat");
    hdk_check(hdk_aa_dots(&dv_, ctl_, qhat_, qcur_, lastq_, lastg_, dq_, dg_, part_b_, s), "aa dots");
    hdk_check(hdk_aa_solve(ctl_, part_b_, 0, s), "aa solve");
    hdk_check(hdk_aa_mix(&dv_, ctl_, qhat_, qcur_, qprev_, q_, dq_, dg_, part_c_, 0, s), "aa mix");
    hdk_check(hdk_gate(ctl_, part_a_, part_c_, 0ULL, s), "gate");
    kernel_launches += 18;
    ++solve_count;
    cuda_check(cudaMemcpyAsync(&host_info, cinfo_, sizeof(int), cudaMemcpyDeviceToHost, st_), "info");
    sync_ctl();
    if (host_info != 0)
      raise(Code::SingularContactSystem, "forward step: contact system is singular even after the diagonal lift");
    if (!h_ctl_->cond) break;
  }
}

// One reverse step for recorded frame t (backward.cpp:396-414); the frame's
// data is already in the working buffers.
void Engine::backward_frame(int t, GradOut& out) {
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  const Frame& f = slots_[t];
  phase_mark(3);
  cuda_check(cudaGraphLaunch(bpre_, st_), "backward pre");
  phase_mark(4);
  run_graph(*bgraph_, "backbone");
  phase_mark(5);
  sync_ctl();
  check_ctl("backward step");
  int iters = 1 + h_ctl_->iterations;  // the first solve of the backbone counts (backward.cpp:176-178)
  last_backward_iterations_ = h_ctl_->iterations;
  kernel_launches += bk_pre_ + static_cast<long long>(bk_body_) * ((h_ctl_->iterations + unroll_ - 1) / unroll_);
  out.tau[t] = h_ctl_->tau;
  out.rho[t] = h_ctl_->rho;
  ContactFrame* c = f.contacts && f.contacts->k > 0 ? f.contacts.get() : nullptr;
  if (c) {
    const int k = c->k;
    if (cX_cols_ < static_cast<size_t>(k)) {
      if (cX_) cudaFree(cX_);
      cuda_check(cudaMalloc(&cX_, sizeof(double) * n3 * k), "contact columns");
      cX_cols_ = k;
    }
    if (!cz0_) cuda_check(cudaMalloc(&cz0_, sizeof(double) * n3), "z0");
    cuda_check(cudaMemcpyAsync(cz0_, x_, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st_), "z0");
    // tangent columns x_c = (A - B)^{-1} j_c warm-started from a_c (backward.cpp:229-238),
    // kColumns at a time through one multi-column stream of the factor
    for (int r = 0; r < k; r += kColumns) iters += solve_columns(*c, r);
    ensure_solver_workspace(k);
    auto hnd = static_cast<cusolverDnHandle_t>(cusolver_);
    hdk_check(hdk_contact_reduced(&c->view, cX_, n3, c->omega, c->e_diag, cz0_, cM_, crhs_, st_), "reduced");
    sol_check(cusolverDnDpotrf(hnd, CUBLAS_FILL_MODE_LOWER, k, cM_, k, cwork_, cwork_len_, cinfo_), "potrf");
    sol_check(cusolverDnDpotrs(hnd, CUBLAS_FILL_MODE_LOWER, k, 1, cM_, k, crhs_, k, cinfo_), "potrs");
    hdk_check(hdk_contact_combine(static_cast<int>(n3), cz0_, cX_, n3, k, c->omega, crhs_, x_, &ctl_->err, st_),
              "mu");
    kernel_launches += 2;
    sync_ctl();
    check_ctl("backward step");
  }
  cuda_check(cudaGraphLaunch(bpost_a_, st_), "backward post");
  if (c) {
    hdk_check(hdk_contact_friction_pushback(&c->view, c->omega, crhs_, dlq_, st_), "friction pushback");
    ++kernel_launches;
  }
  cuda_check(cudaGraphLaunch(bpost_b_, st_), "backward post");
  phase_mark(6);
  kernel_launches += bk_post_;
  ++a_spmv_count;
  solve_count += iters;
  out.adjoint_iterations += iters;
  sync_ctl();
  phase_collect(3, 6);
  check_ctl("backward step");
}

// Simulate-driver diagnostics (drivers.cpp:101-111, 147-159), read on the
// host after a step.
double Engine::last_fb_residual() const {
  const ContactFrame* c = cur_contacts_.get();
  if (!c || c->nc == 0) return 0.0;
  const Vec q = positions();
  Vec lam(c->k);
  cuda_check(cudaMemcpyAsync(lam.data(), c->lambda, c->k * sizeof(double), cudaMemcpyDeviceToHost, st_), "lambda");
  cuda_check(cudaStreamSynchronize(st_), "lambda");
  double worst = 0;
  for (int i = 0; i < c->nc; ++i) {
    const int v = c->vertex[i];
    const double delta = c->normal[3 * i] * q[3 * v] + c->normal[3 * i + 1] * q[3 * v + 1] +
                         c->normal[3 * i + 2] * q[3 * v + 2] - c->gap[i];
    const double r = c->r_n[i], l = lam[i];
    worst = std::max(worst, std::fabs(delta + r * l - std::sqrt(delta * delta + r * r * l * l)));
  }
  return worst;
}

double Engine::penetration() const {
  if (scene_.obstacles.empty()) return 0.0;
  const Vec q = positions();
  double pen = 0;
  for (const Obstacle& ob : scene_.obstacles)
    for (int v = 0; v < scene_.mesh.nv; ++v) pen = std::max(pen, -signed_distance(ob, {q[3 * v], q[3 * v + 1], q[3 * v + 2]}));
  return pen;
}

}  // namespace hdb
