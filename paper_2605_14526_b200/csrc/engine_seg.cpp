// Lockstep batch of one GPU's system-ID samples ("batched
// kernels process a GPU's samples in one launch (concatenated element and
// vertex index spaces, per-sample S in one CSR pool)").
//
// S copies of one mesh become one problem with concatenated vertex, element
// and elimination index spaces.  The global operator is block diagonal, so
// the factor is too: the copies' S' blocks are one tile-major stream and
// each solve pass streams every sample's factor in one launch.  Element and
// vertex kernels (local step, gathers, B apply, routing) run on the
// concatenation unchanged; prox means and tau are looked up per sample
// (hdk_material::seg_means).  What must stay per sample — the Anderson dots
// and coefficient solves, the dual gate, the trust-region ratio, the
// adjoint convergence test — runs through the hdk_seg_* launchers with the
// sample in blockIdx.y and one hdk_ctl per sample, so every sample follows
// the reference's per-sample algorithm (forward.cpp:148-272,
// backward.cpp:170-204) and stops at its own iteration count; the WHILE
// nodes run while any sample is still iterating, and a finished sample's
// kernels return at once.
#include <algorithm>
#include <cstring>

#include "engine.hpp"

namespace hdb {

namespace {
void hdk_check_s(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }
}  // namespace

Scene make_segmented_scene(const Scene& s, int samples, const double* young) {
  if (samples < 1) raise(Code::InvalidArgument, "segmented batch: at least one sample");
  if (!s.obstacles.empty() || !s.fixed.empty() || s.hook)
    raise(Code::InvalidArgument, "segmented batch: contact-free scenes without Dirichlet vertices or hooks (C5)");
  const Mesh& m = s.mesh;
  const int nv = m.nv, ne = m.ne;
  Scene c;
  c.name = s.name + " x" + std::to_string(samples);
  Mesh& cm = c.mesh;
  cm.nv = nv * samples;
  cm.ne = ne * samples;
  cm.total_volume = m.total_volume * samples;
  cm.topology = m.topology;
  for (int k = 0; k < samples; ++k) {
    cm.rest.insert(cm.rest.end(), m.rest.begin(), m.rest.end());
    for (const auto& e : m.el) cm.el.push_back({e[0] + k * nv, e[1] + k * nv, e[2] + k * nv, e[3] + k * nv});
    cm.bm.insert(cm.bm.end(), m.bm.begin(), m.bm.end());
    cm.vol.insert(cm.vol.end(), m.vol.begin(), m.vol.end());
    cm.mass.insert(cm.mass.end(), m.mass.begin(), m.mass.end());
    for (int b : m.boundary) cm.boundary.push_back(b + k * nv);
  }
  Material& mat = c.material;
  mat = s.material;
  mat.young.clear();
  mat.mu.clear();
  mat.lambda.clear();
  mat.beta.clear();
  mat.seg_means.clear();
  for (int k = 0; k < samples; ++k) {
    Material mk = s.material;
    if (young) mk.set_young(Vec(young + static_cast<size_t>(k) * ne, young + static_cast<size_t>(k + 1) * ne), m.vol);
    mat.young.insert(mat.young.end(), mk.young.begin(), mk.young.end());
    mat.mu.insert(mat.mu.end(), mk.mu.begin(), mk.mu.end());
    mat.lambda.insert(mat.lambda.end(), mk.lambda.begin(), mk.lambda.end());
    mat.beta.insert(mat.beta.end(), mk.beta.begin(), mk.beta.end());  // beta_e uses the copy's own max mu
    mat.seg_means.insert(mat.seg_means.end(), {mk.mu_bar, mk.lambda_bar, mk.k_bar});
  }
  c.gravity = s.gravity;
  for (int k = 0; k < samples; ++k) {
    if (!s.f_extra.empty()) c.f_extra.insert(c.f_extra.end(), s.f_extra.begin(), s.f_extra.end());
    c.q0.insert(c.q0.end(), s.q0.begin(), s.q0.end());
    c.v0.insert(c.v0.end(), s.v0.begin(), s.v0.end());
  }
  c.solver = s.solver;
  c.frames = s.frames;
  c.ordering = s.ordering;
  return c;
}

// New moduli for every copy (young: the concatenation): each copy's weights,
// damping and — unless frozen — prox means are its own (material.cpp:48-73).
void segmented_set_young(Material& mat, const Vec& young, const Vec& vol, int samples) {
  const size_t ne = young.size() / samples;
  if (young.size() != mat.young.size() || ne * samples != young.size())
    raise(Code::Validation, "set_young: element count mismatch");
  const Vec vol1(vol.begin(), vol.begin() + ne);
  std::vector<std::uint64_t> versions(samples);
  // samples are independent slices: one host thread per group of samples
  parallel_ranges(
      samples,
      [&](long long k0, long long k1) {
        for (long long k = k0; k < k1; ++k) {
          Material mk;  // the copy's scalars and its slices (not the whole concatenation)
          mk.kind = mat.kind;
          mk.barrier = mat.barrier;
          mk.poisson = mat.poisson;
          mk.alpha = mat.alpha;
          mk.beta0 = mat.beta0;
          mk.frozen = mat.frozen;
          mk.young.assign(mat.young.begin() + k * ne, mat.young.begin() + (k + 1) * ne);
          if (mat.frozen) {
            mk.mu_bar = mat.seg_means[3 * k];
            mk.lambda_bar = mat.seg_means[3 * k + 1];
            mk.k_bar = mat.seg_means[3 * k + 2];
          }
          mk.set_young(Vec(young.begin() + k * ne, young.begin() + (k + 1) * ne), vol1);
          std::copy(mk.young.begin(), mk.young.end(), mat.young.begin() + k * ne);
          std::copy(mk.mu.begin(), mk.mu.end(), mat.mu.begin() + k * ne);
          std::copy(mk.lambda.begin(), mk.lambda.end(), mat.lambda.begin() + k * ne);
          std::copy(mk.beta.begin(), mk.beta.end(), mat.beta.begin() + k * ne);
          mat.seg_means[3 * k] = mk.mu_bar;
          mat.seg_means[3 * k + 1] = mk.lambda_bar;
          mat.seg_means[3 * k + 2] = mk.k_bar;
          versions[k] = mk.version;
        }
      },
      0, 1);
  mat.version = *std::max_element(versions.begin(), versions.end());
}

// Host OR of the samples' loop conditions after sync_ctl (host-driven loops).
bool Engine::host_any() const {
  for (int k = 0; k < segs_; ++k)
    if (h_ctl_[k].cond && h_ctl_[k].err == 0 && h_ctl_[k].nonfinite == 0) return true;
  return false;
}

void Engine::build_forward_graph_seg() {
  const Solver& so = scene_.solver;
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  const double h = so.h;
  void* s = st_;
  auto pre = [&] {
    hdk_check_s(hdk_seg_ctl_init(ctl_, &dseg_, seg_windows_, 10.0, so.k_max, so.eps_rel, so.eps_abs, 0.0, eps_tr_, any_,
                                 s), "ctl init");
    hdk_check_s(hdk_free_fall(&dv_, q_, v_, fext_, h, -1, nullptr, qtil_, qcur_, s), "free fall");
    if (dmat_.beta_vh) hdk_check_s(hdk_damping_elements(&dm_, dmat_.beta_vh, q_, ef2_, s), "damping elements");
    hdk_check_s(hdk_gather(&dv_, dmat_.beta_vh ? ef2_ : nullptr, mat_.alpha / h, q_, nullptr, damp_, s), "damping gather");
    cuda_check(cudaMemcpyAsync(qhat_, q_, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st_), "qhat init");
  };
  auto body = [&](unsigned long long handle) {
    hdk_check_s(hdk_local_step_seg(&dm_, &dmat_, qcur_, ef_, &ctl_->err, ctl_, corner_vpos_, s), "local step");
    hdk_check_s(hdk_seg_gather_rhs_sorted(&dv_, &dseg_, ctl_, ef_, 1.0 / (h * h), qtil_, damp_, bprev_, rhs_, part_a_, s), "rhs");
    hdk_check_s(hdk_apply_inverse3_partial(&df_, rhs_, s), "solve");
    hdk_check_s(hdk_seg_aa_dots_fused(&dv_, &df_, &dseg_, ctl_, qhat_, qcur_, lastq_, lastg_, dq_, dg_, part18_, ticket_,
                                      s), "aa dots + solve");
    hdk_check_s(hdk_seg_aa_mix(&dv_, &dseg_, ctl_, qhat_, qcur_, qprev_, dq_, dg_, part_c_, s), "aa mix");
    hdk_check_s(hdk_seg_gate(ctl_, &dseg_, part_a_, part_c_, any_, gate_ticket_, handle, s), "gate");
  };
  auto post = [&] {
    hdk_check_s(hdk_local_step(&dm_, &dmat_, qcur_, ef_, cache_, &ctl_->err, s), "cache sweep");
  };
  build_loop_graph(st_, use_cond_, pre, body, post, *fgraph_);
  fk_pre_ = fgraph_->counts[0];
  fk_body_ = fgraph_->counts[1];
  fk_post_ = fgraph_->counts[2];
}

void Engine::build_backward_graph_seg() {
  const Solver& so = scene_.solver;
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  const double h = so.h;
  const double umu = 1.0 / (2.0 * (1.0 + mat_.poisson));  // lame(1, nu) (backward.cpp:363)
  const double ula = mat_.poisson / ((1.0 + mat_.poisson) * (1.0 - 2.0 * mat_.poisson));
  void* s = st_;
  for (cudaGraphExec_t* e : {&bpre_, &bpost_a_, &bpost_b_})
    if (*e) {
      cudaGraphExecDestroy(*e);
      *e = nullptr;
    }
  const auto capture = [&](const std::function<void()>& fn, int* kernels) {
    cudaGraph_t g = nullptr;
    cuda_check(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal), "begin capture");
    fn();
    cuda_check(cudaStreamEndCapture(st_, &g), "end capture");
    size_t nn = 0;
    cuda_check(cudaGraphGetNodes(g, nullptr, &nn), "graph nodes");
    if (kernels) *kernels = static_cast<int>(nn);
    cudaGraphExec_t e = nullptr;
    cuda_check(cudaGraphInstantiate(&e, g, 0), "instantiate");
    cudaGraphDestroy(g);
    return e;
  };
  // tr_select_tau per sample, differential with each sample's tau, seed and the first solve
  bpre_ = capture([&] {
    hdk_check_s(hdk_seg_ctl_init(ctl_, &dseg_, seg_windows_ + segs_, 1e8, 500, 0.0, 0.0, 1e-10, eps_tr_, any_, s),
                "ctl init");
    hdk_check_s(hdk_seg_tr_model(&dv_, &dseg_, &a_ff_, bqstar_, bqprev_, dqp_, part_a_, s), "tr model");
    hdk_check_s(hdk_element_energy2(&dm_, &dmat_, bqprev_, eprev_, bqstar_, estar_, &ctl_->bad, s), "energies");
    hdk_check_s(hdk_seg_tr_select(&dv_, &dseg_, eprev_, estar_, bqprev_, bqstar_, bqtil_, 1.0 / (h * h), part_a_,
                                  part_b_, ctl_, s), "tr select");
    hdk_check_s(hdk_differential(&dm_, &dmat_, bcache_, &ctl_->tau, dcomp_, &ctl_->err, s), "differential");
    hdk_check_s(hdk_axpby(static_cast<int>(n3), 1.0, qbar_, 1.0 / h, vbar_, seed_, s), "seed");
    cuda_check(cudaMemsetAsync(x_, 0, n3 * sizeof(double), st_), "x zero");
    cuda_check(cudaMemsetAsync(t_, 0, n3 * sizeof(double), st_), "t zero");
    hdk_check_s(hdk_gather_perm(&dv_, seed_, nullptr, rhs_, s), "x0 rhs");
    hdk_check_s(hdk_apply_inverse3(&df_, rhs_, x_, s), "x0 solve");
  }, &bk_pre_);
  auto pre = [&] {
    hdk_check_s(hdk_seg_aa_reset(ctl_, &dseg_, HDK_AA_MAX, 1e8, 500, 1e-10, any_, s), "aa reset");
    hdk_check_s(hdk_gather_perm(&dv_, seed_, nullptr, seedp_, s), "seed in elimination order");
    hdk_check_s(hdk_gather_perm(&dv_, x_, nullptr, xp_, s), "x0 in elimination order");
    hdk_check_s(hdk_bapply(&dm_, dcomp_, x_, ef_, s), "B x0");
    hdk_check_s(hdk_gather_pp(&dv_, nullptr, ef_, rx_, nullptr, s), "R(x0)");
    hdk_check_s(hdk_axpby(3 * hf_.n, 1.0, seedp_, 1.0, rx_, rhs_, s), "rhs0");
  };
  auto body = [&](unsigned long long handle) {
    for (int u = 0; u < unroll_; ++u) backbone_body_seg(handle);
  };
  build_loop_graph(st_, use_cond_, pre, body, [] {}, *bgraph_);
  bk_body_ = bgraph_->counts[1];
  bk_pre_ += bgraph_->counts[0];
  bpost_a_ = capture([&] {
    hdk_check_s(hdk_route_elements(&dm_, &dmat_, bcache_, bqstar_, x_, umu, ula, dlw_, dle_,
                                   dmat_.beta_vh ? ef2_ : nullptr, s), "route elements");
    hdk_check_s(hdk_route_vertices(&dv_, x_, dmat_.beta_vh ? ef2_ : nullptr, nullptr, qbar_, vbar_, nullptr, h,
                                   mat_.alpha, -1, 0.0, 0.0, dlq_, dlv_, dfacc_, s), "route vertices");
  }, &bk_post_);
  int kb = 0;
  bpost_b_ = capture([&] {
    hdk_check_s(hdk_axpby(static_cast<int>(n3), 1.0, dlq_, 1.0, direct_, qbar_, s), "next q seed");
    hdk_check_s(hdk_axpby(static_cast<int>(n3), 1.0, dlv_, 0.0, nullptr, vbar_, s), "next v seed");
  }, &kb);
  bk_post_ += kb;
}

// One lockstep backbone iteration of every still-iterating sample:
//   solve(rhs) -> seg dots (t folded per sample) -> { seg coefficient solves || B t, gather }
//   -> seg mix -> any (WHILE condition; the solve / B t run flag).
void Engine::backbone_body_seg(unsigned long long handle) {
  void* s = st_;
  hdk_factor fb = df_;
  fb.run_flag = any_;
  hdk_check_s(hdk_apply_inverse3_partial(&fb, rhs_, s), "solve");
  hdk_check_s(hdk_seg_bb_dots(&df_, &dseg_, ctl_, snap_, t_, tv_, xp_, lastq_, lastg_, dq_, dg_, part18_, s), "aa dots");
  cudaStream_t sb = branch_ ? st2_ : st_;
  if (branch_) {
    cuda_check(cudaEventRecord(ev_fork_, st_), "fork");
    cuda_check(cudaStreamWaitEvent(st2_, ev_fork_, 0), "fork wait");
  }
  hdk_check_s(hdk_seg_bb_solve(ctl_, &dseg_, snap_, part18_, aares_, sb), "aa solve");
  hdk_check_s(hdk_bapply_sorted(&dm_, dcomp_, tv_, ef_, corner_pos_, any_, s), "B t");
  hdk_check_s(hdk_gather_sorted(&dv_, nullptr, ef_, rt_, any_, s), "R(t)");
  if (branch_) {
    cuda_check(cudaEventRecord(ev_join_, st2_), "join");
    cuda_check(cudaStreamWaitEvent(st_, ev_join_, 0), "join wait");
  }
  hdk_check_s(hdk_seg_bb_mix(&df_, &dseg_, ctl_, snap_, aares_, t_, xp_, x_, dq_, rt_, rx_, lrx_, lrg_, rsq_, seedp_,
                             rhs_, s), "aa mix");
  hdk_check_s(hdk_seg_any(ctl_, &dseg_, any_, handle, s), "any");
}

}  // namespace hdb
