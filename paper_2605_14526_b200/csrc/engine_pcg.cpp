// The adjoint backbone by preconditioned conjugate gradients (pcg.cu): the
// same linear system and the same stopping test as the reference's Anderson
// fixed point (backward.cpp:170-204), a Krylov method instead of the
// window-8 mixing.  One iteration: B p (matrix-free, engine layout), A p
// (A_ff SpMV), q = A p - B p, the CG updates, one global solve z = A^{-1} r.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "engine.hpp"

namespace hdb {

namespace {
void hdk_check_p(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }
}  // namespace

void Engine::build_pcg_graph() {
  const size_t n3p = 3 * static_cast<size_t>(hf_.n), n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  if (!pcg_) {
    DevArena& A = *mem_;
    pcg_ = A.alloc<hdk_pcg>(segs_);
    pcg_part_ = A.alloc<double>(segs_ > 1 ? static_cast<size_t>(HDK_SEG_PSTRIDE) * segs_
                                          : std::max<size_t>(4 * HDK_RED_BLOCKS, hdk_cpcg_partial_stride(hf_.n)));
    pcg_ticket_ = A.alloc<unsigned int>(segs_);
    cuda_zero(pcg_ticket_, sizeof(unsigned int) * segs_, "zero ticket");
    for (double** v : {&pr_, &pz_, &pp_, &pq_, &pap_, &prp_}) *v = A.alloc<double>(n3p);
    ppv_ = A.alloc<double>(n3);
    cuda_zero(ppv_, n3 * sizeof(double), "zero pv");  // fixed vertices stay 0
    cuda_check(cudaMallocHost(&h_pcg_, sizeof(hdk_pcg) * segs_), "pinned pcg");
  }
  if (!pgraph_) pgraph_ = std::make_unique<LoopGraph>();
  if (segs_ > 1) {
    build_pcg_graph_seg();
    return;
  }
  void* s = st_;
  const int n = hf_.n;
  hdk_factor fs = df_;
  fs.run_flag = &pcg_->cond;
  // fused stages (default): q = (A - B) p over a grid covering the rows once,
  // and z folded from the solve's tile partials in the r.z kernel (no
  // separate x-fold launch); HETERODYN_PCG_FUSED=0: the first form
  static const bool fused = [] {
    const char* e = std::getenv("HETERODYN_PCG_FUSED");
    return !(e && e[0] == '0');
  }();
  if (fused && df_.tile_cta2) {
    const size_t pst = hdk_cpcg_partial_stride(n);
    auto pre_f = [&] {
      hdk_check_p(hdk_pcg_init(pcg_, 1e-10, 500, s), "pcg init");
      hdk_check_p(hdk_gather_perm(&dv_, seed_, nullptr, seedp_, s), "seed in elimination order");
      hdk_check_p(hdk_gather_perm(&dv_, x_, nullptr, xp_, s), "x0 in elimination order");
      hdk_check_p(hdk_bapply(&dm_, dcomp_, x_, ef_, s), "B x0");
      hdk_check_p(hdk_gather_pp(&dv_, nullptr, ef_, rx_, nullptr, s), "R(x0)");
      hdk_check_p(hdk_pcg_spmv(&a_ff_, xp_, pap_, pcg_, s), "A x0");
      hdk_check_p(hdk_pcg_r0(static_cast<int>(n3p), seedp_, pap_, rx_, pr_, s), "r0");
      hdk_check_p(hdk_apply_inverse3_partial(&fs, pr_, s), "A^-1 r0 (tile partials)");
      hdk_check_p(hdk_cpcg_rz(&fs, 1, pr_, pz_, xp_, pcg_part_, pst, pcg_ticket_, pcg_, s), "z0, rz");
      hdk_check_p(hdk_pcg_p(n, pz_, pp_, ppv_, df_.p2v, pcg_, 0ULL, s), "p");
    };
    auto body_f = [&](unsigned long long handle) {
      hdk_check_p(hdk_bapply_sorted(&dm_, dcomp_, ppv_, ef_, corner_pos_, &pcg_->cond, s), "B p");
      hdk_check_p(hdk_cpcg_apply(&dv_, &a_ff_, 1, ef_, 0, pp_, pq_, pcg_part_, pst, pcg_ticket_, pcg_, s),
                  "q = (A - B) p");
      hdk_check_p(hdk_pcg_xr(static_cast<int>(n3p), xp_, pr_, pp_, pq_, pcg_, s), "x, r");
      hdk_check_p(hdk_apply_inverse3_partial(&fs, pr_, s), "A^-1 r (tile partials)");
      hdk_check_p(hdk_cpcg_rz(&fs, 1, pr_, pz_, xp_, pcg_part_, pst, pcg_ticket_, pcg_, s), "z, rz");
      hdk_check_p(hdk_pcg_p(n, pz_, pp_, ppv_, df_.p2v, pcg_, handle, s), "p + cond");
    };
    build_loop_graph(st_, use_cond_, pre_f, body_f, [] {}, *pgraph_);
    return;
  }
  auto pre = [&] {
    hdk_check_p(hdk_pcg_init(pcg_, 1e-10, 500, s), "pcg init");
    hdk_check_p(hdk_gather_perm(&dv_, seed_, nullptr, seedp_, s), "seed in elimination order");
    hdk_check_p(hdk_gather_perm(&dv_, x_, nullptr, xp_, s), "x0 in elimination order");
    hdk_check_p(hdk_bapply(&dm_, dcomp_, x_, ef_, s), "B x0");
    hdk_check_p(hdk_gather_pp(&dv_, nullptr, ef_, rx_, nullptr, s), "R(x0)");
    hdk_check_p(hdk_pcg_spmv(&a_ff_, xp_, pap_, pcg_, s), "A x0");
    hdk_check_p(hdk_pcg_r0(static_cast<int>(n3p), seedp_, pap_, rx_, pr_, s), "r0");
    hdk_check_p(hdk_apply_inverse3_perm(&fs, pr_, pz_, s), "z0 = A^-1 r0");
    hdk_check_p(hdk_pcg_rz(static_cast<int>(n3p), pr_, pz_, xp_, pcg_part_, pcg_ticket_, pcg_, s), "rz");
    hdk_check_p(hdk_pcg_p(n, pz_, pp_, ppv_, df_.p2v, pcg_, 0ULL, s), "p");
  };
  // B p, then one fused launch for gather(B p), A p, q and alpha
  auto body = [&](unsigned long long handle) {
    hdk_check_p(hdk_bapply_sorted(&dm_, dcomp_, ppv_, ef_, corner_pos_, &pcg_->cond, s), "B p");
    hdk_check_p(hdk_pcg_apply(&dv_, &a_ff_, ef_, pp_, pq_, pcg_part_, pcg_ticket_, pcg_, s), "q = (A - B) p");
    hdk_check_p(hdk_pcg_xr(static_cast<int>(n3p), xp_, pr_, pp_, pq_, pcg_, s), "x, r");
    hdk_check_p(hdk_apply_inverse3_perm(&fs, pr_, pz_, s), "z = A^-1 r");
    hdk_check_p(hdk_pcg_rz(static_cast<int>(n3p), pr_, pz_, xp_, pcg_part_, pcg_ticket_, pcg_, s), "rz");
    hdk_check_p(hdk_pcg_p(n, pz_, pp_, ppv_, df_.p2v, pcg_, handle, s), "p + cond");
  };
  build_loop_graph(st_, use_cond_, pre, body, [] {}, *pgraph_);
}

// Lockstep batch: one CG per sample, every stage one launch for all samples
// (hdk_spcg_*); the solve runs while any sample iterates.
void Engine::build_pcg_graph_seg() {
  const size_t n3p = 3 * static_cast<size_t>(hf_.n);
  void* s = st_;
  const int S = segs_, ns = dseg_.n, n3s = 3 * dseg_.n, n3 = static_cast<int>(n3p);
  hdk_factor fs = df_;
  fs.run_flag = any_;
  auto pre = [&] {
    hdk_check_p(hdk_spcg_init(pcg_, S, 1e-10, 500, any_, s), "pcg init");
    hdk_check_p(hdk_gather_perm(&dv_, seed_, nullptr, seedp_, s), "seed in elimination order");
    hdk_check_p(hdk_gather_perm(&dv_, x_, nullptr, xp_, s), "x0 in elimination order");
    hdk_check_p(hdk_bapply(&dm_, dcomp_, x_, ef_, s), "B x0");
    hdk_check_p(hdk_gather_pp(&dv_, nullptr, ef_, rx_, nullptr, s), "R(x0)");
    hdk_check_p(hdk_spcg_spmv(&a_ff_, ns, xp_, pap_, pcg_, s), "A x0");
    hdk_check_p(hdk_pcg_r0(n3, seedp_, pap_, rx_, pr_, s), "r0");
    hdk_check_p(hdk_apply_inverse3_perm(&fs, pr_, pz_, s), "z0 = A^-1 r0");
    hdk_check_p(hdk_spcg_rz(n3s, S, pr_, pz_, xp_, pcg_part_, pcg_ticket_, pcg_, s), "rz");
    hdk_check_p(hdk_spcg_p(n3s, n3, pz_, pp_, ppv_, df_.p2v, pcg_, S, any_, 0ULL, s), "p");
  };
  auto body = [&](unsigned long long handle) {
    hdk_check_p(hdk_bapply_sorted(&dm_, dcomp_, ppv_, ef_, corner_pos_, any_, s), "B p");
    hdk_check_p(hdk_spcg_apply(&dv_, &a_ff_, ns, S, ef_, pp_, pq_, pcg_part_, pcg_ticket_, pcg_, s), "q = (A - B) p");
    hdk_check_p(hdk_spcg_xr(n3s, n3, xp_, pr_, pp_, pq_, pcg_, s), "x, r");
    hdk_check_p(hdk_apply_inverse3_perm(&fs, pr_, pz_, s), "z = A^-1 r");
    hdk_check_p(hdk_spcg_rz(n3s, S, pr_, pz_, xp_, pcg_part_, pcg_ticket_, pcg_, s), "rz");
    hdk_check_p(hdk_spcg_p(n3s, n3, pz_, pp_, ppv_, df_.p2v, pcg_, S, any_, handle, s), "p + any");
  };
  build_loop_graph(st_, use_cond_, pre, body, [] {}, *pgraph_);
}

bool Engine::run_pcg(int& iterations) {
  if (!pgraph_ || (!pgraph_->exec && !pgraph_->body)) build_pcg_graph();
  LoopGraph& g = *pgraph_;
  if (g.exec) {
    cuda_check(cudaGraphLaunch(g.exec, st_), "pcg");
  } else {  // host-driven loop (profiling fallback)
    if (g.pre) cuda_check(cudaGraphLaunch(g.pre, st_), "pcg");
    for (;;) {
      cuda_check(cudaMemcpyAsync(h_pcg_, pcg_, sizeof(hdk_pcg) * segs_, cudaMemcpyDeviceToHost, st_), "pcg state");
      cuda_check(cudaStreamSynchronize(st_), "pcg");
      bool on = false;
      for (int k = 0; k < segs_; ++k) on = on || (h_pcg_[k].cond && h_pcg_[k].err == 0);
      if (!on) break;
      cuda_check(cudaGraphLaunch(g.body, st_), "pcg");
    }
  }
  cuda_check(cudaMemcpyAsync(h_pcg_, pcg_, sizeof(hdk_pcg) * segs_, cudaMemcpyDeviceToHost, st_), "pcg state");
  cuda_check(cudaStreamSynchronize(st_), "pcg");
  int most = 0;
  for (int k = 0; k < segs_; ++k) {
    const hdk_pcg& h = h_pcg_[k];
    if (h.err == -1) {  // not positive definite along a direction: the reference's Anderson loop (all samples)
      ++pcg_fallbacks;
      return false;
    }
    if (h.err != 0)
      raise(Code::AdjointDiverged, "backward step: adjoint CG did not settle (cap or non-finite values)" +
                                       (segs_ > 1 ? " in sample " + std::to_string(k) : std::string()));
    most = std::max(most, h.iter);
    if (segs_ > 1) seg_sample_iterations += 1 + h.iter;
  }
  hdk_check_p(hdk_pcg_final(hf_.n, xp_, pz_, x_, df_.p2v, st_), "x = x + z");
  iterations = 1 + most;  // the first solve x0 = A^{-1} s and one solve per CG step (the slowest sample)
  kernel_launches += g.counts[0] + static_cast<long long>(g.counts[1]) * most + 2;
  return true;
}

}  // namespace hdb
