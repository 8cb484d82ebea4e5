// Contact path of the device engine and the per-frame adjoint driver.
//
// Forward (forward.cpp:148-272 with contact.cpp): one CUDA graph per step,
//   setup  — free-fall target, damping, then hdk_contact_setup: detection at
//            q~ in the reference's vertex-major / obstacle-minor order,
//            order-preserving compaction, geometry, frictional list,
//            unique-vertex rows, zero multipliers (one CTA);
//   WHILE  — scalar inverse columns U = A_s^{-1} E of the contact vertices,
//            three unit spikes per 3-axis solve (factor.cpp:237-289);
//   Delassus W and the r_n / r_f stamps (forward.cpp:178-193);
//   WHILE  — the PD loop with the multiplier update inside every iteration
//            (forward.cpp:222-250): local step, rhs, solve, hdk_contact_ncp
//            (weights, lifted system, dense LDL^T, projection), corrected
//            iterate, Anderson mix, dual gate;
//   post   — cache sweep and the converged weights (forward.cpp:258-262).
// The host reads the control block and the contact counts once per step.
// Capacities are grown (and the step re-run; nothing is committed) when a
// step finds more contacts than the working set holds.
//
// Backward (backward.cpp:208-284): the backbone adjoint z0, one warm-started
// backbone per contact row (engine_columns.cpp), the reduced multiplier
// system (LDL^T on the device) and the friction pushback.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstring>

#include "engine.hpp"

#include <cstdlib>

namespace hdb {

namespace {
void hdk_check(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }
inline double dot(P3 a, P3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline P3 sub(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
double signed_distance(const Obstacle& o, P3 x) {
  if (o.kind == 0) return dot(o.normal, x) - o.offset;
  const P3 d = sub(x, o.center);
  return std::sqrt(dot(d, d)) - o.radius;
}
constexpr int kTraceIters = 20000;  // per-iteration patterns kept for at most this many iterations
}  // namespace

ContactFrame::~ContactFrame() {
  if (base) cudaFree(base);
}

void ContactFrame::allocate(int cap_c, int cap_k, int cap_u, int n) {
  if (base && view.cap_c == cap_c && view.cap_k == cap_k && view.cap_u == cap_u && view.n == n) return;
  if (base) cudaFree(base);
  base = nullptr;
  bytes = hdk_contact_block_bytes(cap_c, cap_k, cap_u, n);
  cuda_check(cudaMalloc(&base, bytes), "contact block");
  cuda_zero(base, bytes, "contact block");
  hdk_contact_block_layout(base, cap_c, cap_k, cap_u, n, &view);
}

void Engine::ensure_contact_capacity(int need_c, int need_k, int need_u) {
  const hdk_contacts& v = cw_.view;
  if (cw_.base && need_c <= v.cap_c && need_k <= v.cap_k && need_u <= v.cap_u) return;
  // generous growth: every growth re-captures the graph and re-runs a step
  const int cap_c = std::max({v.cap_c, 2 * need_c, 32});
  const int cap_u = std::max({v.cap_u, 2 * need_u, 32});
  int cap_k = std::max({v.cap_k, cap_c, 2 * need_k});
  const int smem_rows = hdk_contact_smem_rows();
  if (need_k <= smem_rows && cap_k > smem_rows) cap_k = std::max(smem_rows, cap_c);  // keep the system in shared memory
  cw_.allocate(cap_c, cap_k, cap_u, hf_.n);
  if (!h_cnt_) cuda_check(cudaMallocHost(&h_cnt_, sizeof(int) * HDK_CNT_INTS), "pinned counts");
  const size_t ms = std::max(hdk_contact_scratch_doubles(cap_k), static_cast<size_t>(1));
  if (ms > cM_len_) {
    if (cM_) cudaFree(cM_);
    cuda_check(cudaMalloc(&cM_, ms * sizeof(double)), "contact system scratch");
    cM_len_ = ms;
  }
  if (ctr_mem_) cudaFree(ctr_mem_);
  ctr_.cap = std::min(scene_.solver.k_max, kTraceIters);
  const size_t tb = static_cast<size_t>(ctr_.cap) * cap_c;
  cuda_check(cudaMalloc(&ctr_mem_, 2 * tb * sizeof(double)), "contact trace");
  ctr_.clamp = static_cast<double*>(ctr_mem_);
  ctr_.cone = ctr_.clamp + tb;
  build_contact_graph();
}

void Engine::build_contact_graph() {
  const Solver& so = scene_.solver;
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  const double h = so.h;
  const double hk[5] = {scene_.hook_anchor.x, scene_.hook_anchor.y, scene_.hook_anchor.z, scene_.hook_k, scene_.hook_d};
  const int no = static_cast<int>(scene_.obstacles.size());
  void* s = st_;
  const hdk_contacts* cv = &cw_.view;
  std::vector<SeqGraph::Seg> segs(5);
  // free-fall target, damping, detection and contact rows (forward.cpp:162-176, 208)
  segs[0].fn = [&, cv, no](unsigned long long) {
    hdk_check(hdk_ctl_init(ctl_, aa_window_, 10.0, so.k_max, so.eps_rel, so.eps_abs, 0.0, so.eps_tr, 0, s), "ctl init");
    hdk_check(hdk_free_fall(&dv_, q_, v_, fext_, h, scene_.hook ? scene_.hook_vertex : -1, scene_.hook ? hk : nullptr,
                            qtil_, qcur_, s), "free fall");
    if (dmat_.beta_vh) hdk_check(hdk_damping_elements(&dm_, dmat_.beta_vh, q_, ef2_, s), "damping elements");
    hdk_check(hdk_gather(&dv_, dmat_.beta_vh ? ef2_ : nullptr, mat_.alpha / h, q_, nullptr, damp_, s), "damping gather");
    if (!hf_.fixed.empty()) hdk_check(hdk_fixed_coupling(&a_fd_, d_fixed_, q_, fixc_, s), "fixed coupling");
    cuda_check(cudaMemcpyAsync(qhat_, q_, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st_), "qhat init");
    cuda_check(cudaMemcpyAsync(q0c_, q_, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st_), "q0 init");
  };
  // the setup kernel sets the inverse-column loop's condition: it goes in
  // front of the loop, with the loop's handle (segment 1 captures both)
  segs[1].loop = true;
  segs[1].check_first = true;
  segs[1].flag = cw_.view.cnt + HDK_CNT_SPIKE_COND;
  segs[1].fn = [&, cv](unsigned long long handle) {
    hdk_check(hdk_contact_spikes(cv, rhs_, s), "spikes");
    hdk_check(hdk_apply_inverse3_perm(&df_, rhs_, dqp_, s), "inverse columns");
    hdk_check(hdk_contact_unspike(cv, dqp_, handle, s), "unspike");
  };
  segs[2].fn = [&, cv](unsigned long long) { hdk_check(hdk_contact_delassus(cv, h, s), "delassus"); };
  segs[3].loop = true;
  segs[3].flag = &ctl_->cond;
  segs[3].fn = [&, cv](unsigned long long handle) {
    hdk_check(hdk_local_step(&dm_, &dmat_, qcur_, ef_, nullptr, &ctl_->err, s), "local step");
    hdk_check(hdk_gather_rhs(&dv_, ef_, 1.0 / (h * h), qtil_, damp_, hf_.fixed.empty() ? nullptr : fixc_, bprev_, rhs_,
                             part_a_, s), "rhs");
    hdk_check(hdk_apply_inverse3(&df_, rhs_, q0c_, s), "solve");
    hdk_check(hdk_contact_ncp(cv, qcur_, q_, q0c_, cM_, ctl_, &ctr_, s), "multiplier update");
    hdk_check(hdk_contact_correct(cv, df_.p2v, q0c_, qhat_, s), "q hat");
    hdk_check(hdk_aa_dots(&dv_, ctl_, qhat_, qcur_, lastq_, lastg_, dq_, dg_, part_b_, s), "aa dots");
    hdk_check(hdk_aa_solve(ctl_, part_b_, 0, s), "aa solve");
    hdk_check(hdk_aa_mix(&dv_, ctl_, qhat_, qcur_, qprev_, q_, dq_, dg_, part_c_, 0, s), "aa mix");
    hdk_check(hdk_gate(ctl_, part_a_, part_c_, handle, s), "gate");
  };
  segs[4].fn = [&, cv](unsigned long long) {
    hdk_check(hdk_local_step(&dm_, &dmat_, qcur_, ef_, cache_, &ctl_->err, s), "cache sweep");
    hdk_check(hdk_contact_weights(cv, qcur_, q_, s), "weights star");
  };
  // segment 0 ends with the setup kernel, which sets segment 1's condition
  // (a plain segment receives the handle of the loop after it)
  const double margin = so.contact_margin;
  auto seg0 = segs[0].fn;
  segs[0].fn = [&, seg0, cv, no, margin](unsigned long long next_handle) {
    seg0(0ULL);
    hdk_check(hdk_contact_setup(scene_.mesh.nv, df_.v2p, qtil_, no, obst_, margin, cv, ctl_, next_handle, s),
              "contact setup");
  };
  build_seq_graph(st_, use_cond_, std::move(segs), cgraph_);
  for (int i = 0; i < 5; ++i) fc_kernels_[i] = cgraph_.kernels[i];
}

// One forward step of a scene with obstacles; false when the contact set
// overflowed the capacities (grown here; the caller re-runs the step).
bool Engine::run_contact_step() {
  // first capacity: 128 contacts and a 224-row system (the shared-memory
  // factorization's limit), so a growing contact set (C4 reaches ~70 contacts,
  // 200 rows in five steps) does not re-capture the forward graph and re-run
  // steps mid-trajectory
  if (!cw_.base) ensure_contact_capacity(std::min(64, scene_.mesh.nv), hdk_contact_smem_rows() / 2, 64);
  if (cgraph_.exec) {
    cuda_check(cudaGraphLaunch(cgraph_.exec, st_), "contact forward graph");
  } else {
    // host-driven segments (profiling): one status read per loop iteration
    for (size_t i = 0; i < cgraph_.segs.size(); ++i) {
      const SeqGraph::Seg& g = cgraph_.segs[i];
      if (!g.loop) {
        cuda_check(cudaGraphLaunch(cgraph_.parts[i], st_), "contact forward segment");
        continue;
      }
      int flag = 1;
      const auto read_flag = [&] {
        cuda_check(cudaMemcpyAsync(h_cnt_ + HDK_CNT_INTS - 1, g.flag, sizeof(int), cudaMemcpyDeviceToHost, st_), "flag");
        cuda_check(cudaStreamSynchronize(st_), "flag");
        flag = h_cnt_[HDK_CNT_INTS - 1];
      };
      if (g.check_first) read_flag();
      while (flag) {
        cuda_check(cudaGraphLaunch(cgraph_.parts[i], st_), "contact forward loop");
        read_flag();
      }
    }
  }
  return true;
}

void Engine::contact_trace(std::vector<int>& vertex, std::vector<int>& obstacle, std::vector<double>& clamp,
                           std::vector<double>& cone, int& nc, int& nf, int& iterations) const {
  nc = cur_has_contacts_ ? cw_.nc : 0;
  nf = cur_has_contacts_ ? cw_.nf : 0;
  iterations = cur_has_contacts_ ? trace_iters_ : 0;
  vertex.assign(nc, 0);
  obstacle.assign(nc, 0);
  clamp.assign(static_cast<size_t>(iterations) * nc, 0.0);
  cone.assign(static_cast<size_t>(iterations) * nf, 0.0);
  if (nc == 0) return;
  const size_t cap = cw_.view.cap_c;
  cuda_check(cudaMemcpyAsync(vertex.data(), cw_.view.vertex, sizeof(int) * nc, cudaMemcpyDeviceToHost, st_), "trace");
  cuda_check(cudaMemcpyAsync(obstacle.data(), cw_.view.obstacle, sizeof(int) * nc, cudaMemcpyDeviceToHost, st_), "trace");
  if (iterations) {
    cuda_check(cudaMemcpy2DAsync(clamp.data(), sizeof(double) * nc, ctr_.clamp, sizeof(double) * cap, sizeof(double) * nc,
                                 iterations, cudaMemcpyDeviceToHost, st_), "trace");
    if (nf)
      cuda_check(cudaMemcpy2DAsync(cone.data(), sizeof(double) * nf, ctr_.cone, sizeof(double) * cap,
                                   sizeof(double) * nf, iterations, cudaMemcpyDeviceToHost, st_), "trace");
  }
  cuda_check(cudaStreamSynchronize(st_), "trace");
}

// One reverse step for recorded frame t (backward.cpp:396-414); the frame's
// data is already in the working buffers.
void Engine::backward_frame(int t, GradOut& out) {
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  const Frame& f = slots_[t];
  phase_mark(3);
  cuda_check(cudaGraphLaunch(bpre_, st_), "backward pre");
  phase_mark(4);
  int pcg_iters = -1;
  if (!(use_pcg_ && run_pcg(pcg_iters))) run_graph(*bgraph_, "backbone");
  phase_mark(5);
  sync_ctl();
  check_ctl("backward step");
  int iters = pcg_iters >= 0 ? pcg_iters : 1 + h_ctl_->iterations;  // the first solve counts (backward.cpp:176-178)
  if (segs_ > 1) {  // lockstep: every sample's own count, the loop ran to the largest
    seg_tau.resize(segs_);
    for (int k = 0; k < segs_; ++k) {
      if (pcg_iters < 0) {  // (the CG path counted its samples in run_pcg)
        iters = std::max(iters, 1 + h_ctl_[k].iterations);
        seg_sample_iterations += 1 + h_ctl_[k].iterations;
      }
      seg_tau[k] = h_ctl_[k].tau;
    }
  }
  last_backward_iterations_ = iters - 1;
  kernel_launches += bk_pre_ + static_cast<long long>(bk_body_) * ((h_ctl_->iterations + unroll_ - 1) / unroll_);
  out.tau[t] = h_ctl_->tau;
  out.rho[t] = h_ctl_->rho;
  ContactFrame* c = f.has_contacts && f.contacts->k > 0 ? f.contacts.get() : nullptr;
  if (c) {
    const int k = c->k;
    if (cX_cols_ < static_cast<size_t>(k)) {  // sized to the contact block's row capacity (grown geometrically)
      const size_t cols = std::max(static_cast<size_t>(k), static_cast<size_t>(c->view.cap_k));
      if (cX_) cudaFree(cX_);
      cuda_check(cudaMalloc(&cX_, sizeof(double) * n3 * cols), "contact columns");
      cX_cols_ = cols;
    }
    if (!cz0_) cuda_check(cudaMalloc(&cz0_, sizeof(double) * n3), "z0");
    cuda_check(cudaMemcpyAsync(cz0_, x_, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st_), "z0");
    // tangent columns x_c = (A - B)^{-1} j_c warm-started from a_c (backward.cpp:229-238),
    // kColumns at a time through one multi-column stream of the factor
    static const bool refill = [] {  // opt-in: measured slower
      const char* e = std::getenv("HETERODYN_COLUMN_REFILL");
      return e && e[0] == '1';
    }();
    if (refill) {
      iters += solve_all_columns(*c);
    } else {
      if (use_pcg_) column_deflation_setup();
      for (int r = 0; r < k; r += kColumns) iters += solve_columns(*c, r);
    }
    const size_t ms = hdk_contact_scratch_doubles(c->view.cap_k);
    if (ms > cM_len_) {
      if (cM_) cudaFree(cM_);
      cuda_check(cudaMalloc(&cM_, ms * sizeof(double)), "contact system scratch");
      cM_len_ = ms;
    }
    hdk_check(hdk_contact_reduced(&c->view, cX_, n3, cz0_, cM_, &ctl_->err, st_), "reduced system");
    hdk_check(hdk_contact_combine(&c->view, static_cast<int>(n3), cz0_, cX_, n3, x_, st_), "mu");
    kernel_launches += 2;
    sync_ctl();
    check_ctl("backward step");
  }
  cuda_check(cudaGraphLaunch(bpost_a_, st_), "backward post");
  if (c) {
    hdk_check(hdk_contact_friction_pushback(&c->view, dlq_, st_), "friction pushback");
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
  if (ph_.per_frame) {
    float pre = 0.f, loop = 0.f, post = 0.f;
    cudaEventElapsedTime(&pre, ph_.ev[3], ph_.ev[4]);
    cudaEventElapsedTime(&loop, ph_.ev[4], ph_.ev[5]);
    cudaEventElapsedTime(&post, ph_.ev[5], ph_.ev[6]);
    std::fprintf(stderr, "[frame %d] pre %.3f backbone %.3f post %.3f ms (columns %.3f ms), K %d, iterations %d\n", t,
                 pre, loop, post, ph_.col_ms - ph_.last_col_ms, c ? c->k : 0, iters);
    ph_.last_col_ms = ph_.col_ms;
  }
  check_ctl("backward step");
}

// Simulate-driver diagnostics (drivers.cpp:101-111, 147-159), read on the
// host after a step.
double Engine::last_fb_residual() const {
  if (!cur_has_contacts_ || cw_.nc == 0) return 0.0;
  const int nc = cw_.nc, k = cw_.k;
  const Vec q = positions();
  std::vector<int> vert(nc);
  Vec nrm(3 * static_cast<size_t>(nc)), gap(nc), rn(nc), lam(k);
  const hdk_contacts& c = cw_.view;
  cuda_check(cudaMemcpyAsync(vert.data(), c.vertex, sizeof(int) * nc, cudaMemcpyDeviceToHost, st_), "contacts");
  cuda_check(cudaMemcpyAsync(nrm.data(), c.normal, sizeof(double) * 3 * nc, cudaMemcpyDeviceToHost, st_), "contacts");
  cuda_check(cudaMemcpyAsync(gap.data(), c.gap, sizeof(double) * nc, cudaMemcpyDeviceToHost, st_), "contacts");
  cuda_check(cudaMemcpyAsync(rn.data(), c.r_n, sizeof(double) * nc, cudaMemcpyDeviceToHost, st_), "contacts");
  cuda_check(cudaMemcpyAsync(lam.data(), c.lambda, sizeof(double) * k, cudaMemcpyDeviceToHost, st_), "contacts");
  cuda_check(cudaStreamSynchronize(st_), "contacts");
  double worst = 0;
  for (int i = 0; i < nc; ++i) {
    const int v = vert[i];
    const double delta = nrm[3 * i] * q[3 * v] + nrm[3 * i + 1] * q[3 * v + 1] + nrm[3 * i + 2] * q[3 * v + 2] - gap[i];
    const double r = rn[i], l = lam[i];
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
