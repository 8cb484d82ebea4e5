#include <cmath>
// The adjoint backbone by preconditioned conjugate gradients (pcg.cu): the
// same linear system and the same stopping test as the reference's Anderson
// fixed point (backward.cpp:170-204), a Krylov method instead of the
// window-8 mixing.  One iteration: B p (matrix-free, engine layout), A p
// (A_ff SpMV), q = A p - B p, the CG updates, one global solve z = A^{-1} r.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "engine.hpp"

namespace hdb {

namespace {
void hdk_check_p(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

// The CG's preconditioner solves z = A^{-1} r may stream the fp32 copy of S'
// (hdk_factor::use32): CG converges to the solution of (A - B) x = s for any
// fixed SPD preconditioner, and M = S~^T S~ with S~ the fp32-rounded factor is
// one; its residuals r and the operator applies stay fp64, so x is exact to
// the stopping test and x + z differs from x + A^{-1} r by (M - A^{-1}) r,
// ~1e-7 of a quantity the test has already made 1e-10 of x.  The forward
// solves, the first backbone solve and the contact columns' warm starts keep
// the fp64 factor.  Opt-in (HETERODYN_PCG_FP32=1): the passes are not
// bandwidth-bound at these sizes (C3: 35.9 / 28.4 us with half the bytes vs
// 36.5 / 31.5 us), and the rounded preconditioner costs iterations (C3 36.9 vs
// 34.0 solves per step: 221 vs 230 steps/s; C5 1383 vs 1330 sample-steps/s).
bool pcg_fp32_preconditioner() {
  const char* e = std::getenv("HETERODYN_PCG_FP32");
  return e && e[0] == '1';
}
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
  fs.use32 = pcg_fp32_preconditioner() ? 1 : 0;
  // fused stages (default): q = (A - B) p over a grid covering the rows once,
  // and z folded from the solve's tile partials in the r.z kernel (no
  // separate x-fold launch); HETERODYN_PCG_FUSED=0: the first form
  static const bool fused = [] {
    const char* e = std::getenv("HETERODYN_PCG_FUSED");
    return !(e && e[0] == '0');
  }();
  if (fused && df_.tile_cta2) {
    const size_t pst = hdk_cpcg_partial_stride(n);
    if (defl_.on) defl_alloc();
    Deflation& D = defl_;
    const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv), ne = scene_.mesh.ne;
    const int cstride = static_cast<int>(sizeof(hdk_pcg) / sizeof(int));
    auto pre_f = [&] {
      if (D.on) {
        hdk_check_p(hdk_pcg_init(pcg_, 1e-10, 500, s), "pcg init");
        hdk_check_p(hdk_gather_perm(&dv_, seed_, nullptr, seedp_, s), "seed in elimination order");
        hdk_check_p(hdk_gather_perm(&dv_, x_, nullptr, xp_, s), "x0 in elimination order");
        hdk_check_p(hdk_bapply(&dm_, dcomp_, x_, ef_, s), "B x0");
        hdk_check_p(hdk_gather_pp(&dv_, nullptr, ef_, rx_, nullptr, s), "R(x0)");
        hdk_check_p(hdk_pcg_spmv(&a_ff_, xp_, pap_, pcg_, s), "A x0");
        hdk_check_p(hdk_pcg_r0(static_cast<int>(n3p), seedp_, pap_, rx_, pr_, s), "r0");
        // this step's (A - B) W, E = W^T (A - B) W, and the Galerkin first iterate
        hdk_check_p(hdk_scatter_cols(n, scene_.mesh.nv, HDK_DEFL_MAX, D.w, D.wv, df_.p2v, D.d, s), "W by vertex");
        for (int g = 0; g < HDK_DEFL_MAX; g += 8)  // B W, eight columns per launch
          hdk_check_p(hdk_bapply_cols_sorted(&dm_, dcomp_, D.wv + g * n3, n3, D.ef8 + g * 12 * ne, 12 * ne, corner_pos_,
                                             &D.ones[g].cond, cstride, 8, s),
                      "B W");
        hdk_check_p(hdk_cpcg_apply_q(&dv_, &a_ff_, HDK_DEFL_MAX, D.ef8, 12 * ne, D.w, D.aw, D.ones, s), "(A - B) W");
        hdk_check_p(hdk_defl_gram(static_cast<int>(n3p), D.w, D.aw, D.part, D.ticket, D.d, s), "E = W^T A' W");
        hdk_check_p(hdk_defl_galerkin(static_cast<int>(n3p), xp_, pr_, D.w, D.aw, D.part, D.ticket, D.d, s),
                    "Galerkin first iterate");
        hdk_check_p(hdk_apply_inverse3_partial(&fs, pr_, s), "A^-1 r0 (tile partials)");
        hdk_check_p(hdk_dpcg_rz(&fs, pr_, pz_, xp_, D.aw, D.part, D.ticket, pcg_, D.d, D.zhist, D.hist, s), "z0, rz");
        hdk_check_p(hdk_dpcg_p(n, pz_, pp_, ppv_, df_.p2v, pcg_, D.d, D.w, 0ULL, s), "p");
        return;
      }
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
      if (D.on) {
        hdk_check_p(hdk_dpcg_rz(&fs, pr_, pz_, xp_, D.aw, D.part, D.ticket, pcg_, D.d, D.zhist, D.hist, s), "z, rz");
        hdk_check_p(hdk_dpcg_p(n, pz_, pp_, ppv_, df_.p2v, pcg_, D.d, D.w, handle, s), "p + cond");
        return;
      }
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
  fs.use32 = pcg_fp32_preconditioner() ? 1 : 0;
  if (defl_.on) {  // per-sample recycled deflation (the single engine's scheme, sample by sample)
    defl_alloc();
    Deflation& D = defl_;
    const size_t nvv = 3 * static_cast<size_t>(scene_.mesh.nv), ne = scene_.mesh.ne;
    const int cstride = static_cast<int>(sizeof(hdk_pcg) / sizeof(int));
    auto pre_d = [&] {
      hdk_check_p(hdk_spcg_init(pcg_, S, 1e-10, 500, any_, s), "pcg init");
      hdk_check_p(hdk_gather_perm(&dv_, seed_, nullptr, seedp_, s), "seed in elimination order");
      hdk_check_p(hdk_gather_perm(&dv_, x_, nullptr, xp_, s), "x0 in elimination order");
      hdk_check_p(hdk_bapply(&dm_, dcomp_, x_, ef_, s), "B x0");
      hdk_check_p(hdk_gather_pp(&dv_, nullptr, ef_, rx_, nullptr, s), "R(x0)");
      hdk_check_p(hdk_spcg_spmv(&a_ff_, ns, xp_, pap_, pcg_, s), "A x0");
      hdk_check_p(hdk_pcg_r0(n3, seedp_, pap_, rx_, pr_, s), "r0");
      hdk_check_p(hdk_scatter_cols(hf_.n, scene_.mesh.nv, HDK_DEFL_MAX, D.w, D.wv, df_.p2v, D.d, s), "W by vertex");
      for (int g = 0; g < HDK_DEFL_MAX; g += 8)
        hdk_check_p(hdk_bapply_cols_sorted(&dm_, dcomp_, D.wv + g * nvv, nvv, D.ef8 + g * 12 * ne, 12 * ne,
                                           corner_pos_, &D.ones[g].cond, cstride, 8, s),
                    "B W");
      hdk_check_p(hdk_cpcg_apply_q(&dv_, &a_ff_, HDK_DEFL_MAX, D.ef8, 12 * ne, D.w, D.aw, D.ones, s), "(A - B) W");
      hdk_check_p(hdk_sdefl_gram(n3s, S, D.w, D.aw, D.d, D.ds, D.e, s), "E per sample");
      hdk_check_p(hdk_sdefl_galerkin(n3s, S, xp_, pr_, D.w, D.aw, D.d, D.ds, pcg_part_, D.tickets, s),
                  "Galerkin first iterates");
      hdk_check_p(hdk_apply_inverse3_perm(&fs, pr_, pz_, s), "z0 = A^-1 r0");
      hdk_check_p(hdk_sdpcg_rz(n3s, S, pr_, pz_, xp_, D.aw, pcg_part_, pcg_ticket_, pcg_, D.d, D.ds, D.zhist, D.hist, s),
                  "rz");
      hdk_check_p(hdk_sdpcg_p(n3s, n3, pz_, pp_, ppv_, df_.p2v, pcg_, S, any_, D.d, D.ds, D.w, 0ULL, s), "p");
    };
    auto body_d = [&](unsigned long long handle) {
      hdk_check_p(hdk_bapply_sorted_seg(&dm_, dcomp_, ppv_, ef_, corner_pos_, &pcg_->cond,
                                        static_cast<int>(sizeof(hdk_pcg) / sizeof(int)), dseg_.ne, s), "B p");
      hdk_check_p(hdk_spcg_apply(&dv_, &a_ff_, ns, S, ef_, pp_, pq_, pcg_part_, pcg_ticket_, pcg_, s), "q = (A - B) p");
      hdk_check_p(hdk_spcg_xr(n3s, n3, xp_, pr_, pp_, pq_, pcg_, s), "x, r");
      hdk_check_p(hdk_apply_inverse3_perm(&fs, pr_, pz_, s), "z = A^-1 r");
      hdk_check_p(hdk_sdpcg_rz(n3s, S, pr_, pz_, xp_, D.aw, pcg_part_, pcg_ticket_, pcg_, D.d, D.ds, D.zhist, D.hist, s),
                  "rz");
      hdk_check_p(hdk_sdpcg_p(n3s, n3, pz_, pp_, ppv_, df_.p2v, pcg_, S, any_, D.d, D.ds, D.w, handle, s), "p + any");
    };
    build_loop_graph(st_, use_cond_, pre_d, body_d, [] {}, *pgraph_);
    return;
  }
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
    hdk_check_p(hdk_bapply_sorted_seg(&dm_, dcomp_, ppv_, ef_, corner_pos_, &pcg_->cond,
                                        static_cast<int>(sizeof(hdk_pcg) / sizeof(int)), dseg_.ne, s), "B p");
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
  // profiling: HETERODYN_CG_TRACE1=path writes the (alpha, beta) of the last
  // backbone CG (the fused path's r.z kernel records them)
  static const char* trace1 = std::getenv("HETERODYN_CG_TRACE1");
  static double* d_tr = nullptr;
  static double** h_tr = nullptr;
  if (trace1 && !d_tr) {
    cuda_check(cudaMalloc(&d_tr, sizeof(double) * 8 * 512 * 2), "cg trace");
    cuda_check(cudaMallocHost(&h_tr, 2 * sizeof(double*)), "cg trace");
    h_tr[0] = d_tr;
    h_tr[1] = nullptr;
  }
  if (d_tr) {
    cuda_check(cudaMemsetAsync(d_tr, 0, sizeof(double) * 8 * 512 * 2, st_), "cg trace");
    hdk_check_p(hdk_set_cpcg_trace(h_tr, st_), "cg trace");
  }
  if (defl_.on && defl_.d) {  // this solve: deflate with W, or record the Ritz data for W
    Deflation& D = defl_;
    const bool pause = !D.valid && D.cooldown > 0;
    if (pause) --D.cooldown;
    D.h->use = D.valid ? 1 : 0;
    D.h->k = D.valid ? D.k : 0;
    D.h->rec = (D.valid || pause) ? 0 : 1;
    D.h->hcap = D.hcap;
    D.h->active = 0;
    D.h->cols = 0;
    cuda_check(cudaMemcpyAsync(&D.d->k, &D.h->k, 6 * sizeof(int), cudaMemcpyHostToDevice, st_), "deflation flags");
    for (int c = 0; c < HDK_DEFL_MAX; ++c) D.h_ones[c].cond = (D.valid && c < D.k) ? 1 : 0;
    cuda_check(cudaMemcpyAsync(D.ones, D.h_ones, HDK_DEFL_MAX * sizeof(hdk_pcg), cudaMemcpyHostToDevice, st_),
               "deflation flags");
  }
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
  if (d_tr) {
    hdk_check_p(hdk_set_cpcg_trace(h_tr + 1, st_), "cg trace off");
    std::vector<double> h(8 * 512 * 2);
    cuda_check(cudaMemcpy(h.data(), d_tr, h.size() * sizeof(double), cudaMemcpyDeviceToHost), "cg trace");
    if (FILE* fp = std::fopen(trace1, "wb")) {
      std::fwrite(h.data(), sizeof(double), h.size(), fp);
      std::fclose(fp);
    }
  }
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
  if (defl_.on && defl_.d && segs_ == 1) defl_after_solve(h_pcg_[0].iter, h_pcg_[0].done != 0);
  if (defl_.on && defl_.d && segs_ > 1) defl_after_solve_seg();
  hdk_check_p(hdk_pcg_final(hf_.n, xp_, pz_, x_, df_.p2v, st_), "x = x + z");
  iterations = 1 + most;  // the first solve x0 = A^{-1} s and one solve per CG step (the slowest sample)
  kernel_launches += g.counts[0] + static_cast<long long>(g.counts[1]) * most + 2;
  return true;
}

}  // namespace hdb

namespace hdb {

void Engine::set_deflation(bool on) {
  defl_.valid = false;
  if (on == defl_.on) return;
  defl_.on = on;
  if (pgraph_) {  // the captured graph has or lacks the deflation stages: re-capture
    pgraph_->destroy();
    pgraph_.reset();
  }
}

void Engine::defl_alloc() {
  Deflation& D = defl_;
  if (D.d) return;
  DevArena& A = *mem_;
  const size_t n3p = 3 * static_cast<size_t>(hf_.n), n3 = 3 * static_cast<size_t>(scene_.mesh.nv),
               ne = scene_.mesh.ne;
  D.hcap = segs_ > 1 ? 160 : 200;
  D.d = A.alloc<hdk_defl>(1);
  if (segs_ > 1) {
    D.ds = A.alloc<hdk_sdefl>(segs_);
    D.e = A.alloc<double>(static_cast<size_t>(segs_) * HDK_DEFL_MAX * HDK_DEFL_MAX);
    D.tickets = A.alloc<unsigned int>(segs_);
  }
  constexpr int K = HDK_DEFL_MAX;
  D.ones = A.alloc<hdk_pcg>(K);
  D.w = A.alloc<double>(K * n3p);
  D.aw = A.alloc<double>(K * n3p);
  D.wv = A.alloc<double>(K * n3);
  D.ef8 = A.alloc<double>(K * 12 * ne);
  D.zhist = A.alloc<double>(static_cast<size_t>(D.hcap) * n3p);
  D.hist = A.alloc<double>(3 * static_cast<size_t>(D.hcap) * segs_);
  D.coef = A.alloc<double>(K * static_cast<size_t>(D.hcap) * segs_);
  D.part = A.alloc<double>(std::max(hdk_defl_partial_doubles(hf_.n), hdk_bcg_partial_doubles(hf_.n)));
  D.ticket = A.alloc<unsigned int>(1);
  cuda_check(cudaMallocHost(&D.h, sizeof(hdk_defl)), "pinned deflation");
  cuda_check(cudaMallocHost(&D.h_ones, K * sizeof(hdk_pcg)), "pinned deflation");
  cuda_check(cudaMallocHost(&D.h_hist, 3 * sizeof(double) * D.hcap * segs_), "pinned deflation");
  cuda_check(cudaMallocHost(&D.h_coef, K * sizeof(double) * D.hcap * segs_), "pinned deflation");
  std::memset(D.h, 0, sizeof(hdk_defl));
  std::memset(D.h_ones, 0, K * sizeof(hdk_pcg));
}

namespace {
// Eigen-decomposition of a symmetric m x m matrix (cyclic Jacobi): a is
// destroyed, eigenvalues into ev, eigenvectors into the columns of v.
void jacobi_eigen(std::vector<double>& a, int m, std::vector<double>& ev, std::vector<double>& v) {
  v.assign(static_cast<size_t>(m) * m, 0.0);
  for (int i = 0; i < m; ++i) v[i * m + i] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) off += a[p * m + q] * a[p * m + q];
    if (off < 1e-30) break;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        const double apq = a[p * m + q];
        if (std::fabs(apq) < 1e-300) continue;
        const double theta = (a[q * m + q] - a[p * m + p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < m; ++k) {  // rotate columns p, q
          const double akp = a[k * m + p], akq = a[k * m + q];
          a[k * m + p] = c * akp - s * akq;
          a[k * m + q] = s * akp + c * akq;
        }
        for (int k = 0; k < m; ++k) {  // rotate rows p, q
          const double apk = a[p * m + k], aqk = a[q * m + k];
          a[p * m + k] = c * apk - s * aqk;
          a[q * m + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < m; ++k) {
          const double vkp = v[k * m + p], vkq = v[k * m + q];
          v[k * m + p] = c * vkp - s * vkq;
          v[k * m + q] = s * vkp + c * vkq;
        }
      }
  }
  ev.resize(m);
  for (int i = 0; i < m; ++i) ev[i] = a[i * m + i];
}
}  // namespace

// After a backbone CG: a recording solve yields W (the Ritz vectors of the
// k smallest Ritz values of its Lanczos matrix, from its z's); a deflated
// solve that needed more than 85 % of the recorded solve's iterations (the
// state has drifted) or whose E lost definiteness drops W, so the next
// solve records again.
void Engine::defl_after_solve(int iterations, bool converged) {
  Deflation& D = defl_;
  if (D.valid) {
    ++D.deflated_solves;
    cuda_check(cudaMemcpy(&D.h->active, &D.d->active, sizeof(int), cudaMemcpyDeviceToHost), "deflation state");
    // Keep W while it pays: a deflated solve costs (A - B)W and E up front and
    // 8 more dots / axpys per iteration, so it must save >= 15 % of the
    // recorded solve's iterations (C3: 34 of 53; C1, 5k tets: 22 of 24 does
    // not pay).  A miss drops W (the next solve records afresh, in case the
    // state drifted); two misses in a row pause deflation for 64 solves.
    if (!D.h->active || iterations > (85 * D.plain_iters) / 100) {
      D.valid = false;
      if (++D.misses >= 2) {
        D.cooldown = 64;
        D.misses = 0;
      }
    } else {
      D.misses = 0;
    }
    return;
  }
  if (D.cooldown > 0) return;  // a plain solve during the pause: nothing recorded
  const int J = iterations;  // z_1 .. z_J recorded (rz calls)
  if (!converged || J < 6 || J > D.hcap) return;
  cuda_check(cudaMemcpy(D.h_hist, D.hist, 3 * sizeof(double) * J, cudaMemcpyDeviceToHost), "Ritz history");
  const int m = J - 1;  // Lanczos matrix from (alpha_j, beta_j), j = 1 .. J - 1
  std::vector<double> T(static_cast<size_t>(m) * m, 0.0), ev, Y;
  for (int j = 0; j < m; ++j) {
    const double a = D.h_hist[3 * (j + 1)], b = D.h_hist[3 * (j + 1) + 1];
    const double ap = j > 0 ? D.h_hist[3 * j] : 0.0, bp = j > 0 ? D.h_hist[3 * j + 1] : 0.0;
    if (!(a > 0.0) || !(b >= 0.0)) return;
    T[j * m + j] = 1.0 / a + (j > 0 ? bp / ap : 0.0);
    if (j + 1 < m) T[j * m + j + 1] = T[(j + 1) * m + j] = std::sqrt(b) / a;
  }
  jacobi_eigen(T, m, ev, Y);
  std::vector<int> order(m);
  for (int i = 0; i < m; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int x, int y) { return ev[x] < ev[y]; });
  static const int kmax = [] {  // HETERODYN_DEFLATION_K: recycled vectors (default and cap HDK_DEFL_MAX)
    const char* e = std::getenv("HETERODYN_DEFLATION_K");
    const int v = e ? std::atoi(e) : HDK_DEFL_MAX;
    return std::max(1, std::min(v, HDK_DEFL_MAX));
  }();
  const int k = std::min(kmax, m / 2);
  for (int c = 0; c < k; ++c)
    for (int j = 0; j < m; ++j) {  // v_j = (-1)^j z_{j+1} / sqrt(r_{j+1}.z_{j+1})
      const double rz = D.h_hist[3 * j + 2];
      D.h_coef[c * m + j] = Y[j * m + order[c]] * ((j & 1) ? -1.0 : 1.0) / std::sqrt(rz);
    }
  cuda_check(cudaMemcpyAsync(D.coef, D.h_coef, sizeof(double) * k * m, cudaMemcpyHostToDevice, st_), "Ritz coefficients");
  hdk_check_p(hdk_ritz_combine(3 * hf_.n, D.zhist, D.coef, m, k, D.w, st_), "Ritz vectors");
  D.k = k;
  D.valid = true;
  D.plain_iters = J;
  ++D.refreshes;
}

// The lockstep batch's version: every sample records together and gets its
// own Ritz vectors (in its range of W); k is the smallest over the samples.
void Engine::defl_after_solve_seg() {
  Deflation& D = defl_;
  const int S = segs_;
  int most = 0;
  bool all_conv = true;
  for (int s = 0; s < S; ++s) {
    most = std::max(most, h_pcg_[s].iter);
    all_conv = all_conv && h_pcg_[s].done != 0;
  }
  if (D.valid) {
    ++D.deflated_solves;
    static const bool verbose = std::getenv("HETERODYN_DEFLATION_LOG") != nullptr;
    if (verbose) std::fprintf(stderr, "[deflation] lockstep solve: %d iterations (recorded %d)\n", most, D.plain_iters);
    if (most > (95 * D.plain_iters) / 100) D.valid = false;
    return;
  }
  if (!all_conv || most < 6 || most > D.hcap) return;
  cuda_check(cudaMemcpy(D.h_hist, D.hist, 3 * sizeof(double) * D.hcap * S, cudaMemcpyDeviceToHost), "Ritz history");
  int kmin = HDK_DEFL_MAX, jmax = 0;
  for (int s = 0; s < S; ++s) {
    jmax = std::max(jmax, h_pcg_[s].iter - 1);
    kmin = std::min(kmin, (h_pcg_[s].iter - 1) / 2);
  }
  if (kmin < 1) return;
  std::fill(D.h_coef, D.h_coef + static_cast<size_t>(S) * HDK_DEFL_MAX * jmax, 0.0);
  std::vector<double> T, ev, Y;
  std::vector<int> order;
  for (int s = 0; s < S; ++s) {
    const double* h = D.h_hist + static_cast<size_t>(s) * 3 * D.hcap;
    const int m = h_pcg_[s].iter - 1;
    T.assign(static_cast<size_t>(m) * m, 0.0);
    for (int j = 0; j < m; ++j) {
      const double a = h[3 * (j + 1)], b = h[3 * (j + 1) + 1];
      const double ap = j > 0 ? h[3 * j] : 0.0, bp = j > 0 ? h[3 * j + 1] : 0.0;
      if (!(a > 0.0) || !(b >= 0.0)) return;
      T[j * m + j] = 1.0 / a + (j > 0 ? bp / ap : 0.0);
      if (j + 1 < m) T[j * m + j + 1] = T[(j + 1) * m + j] = std::sqrt(b) / a;
    }
    jacobi_eigen(T, m, ev, Y);
    order.resize(m);
    for (int i = 0; i < m; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return ev[x] < ev[y]; });
    double* cs = D.h_coef + static_cast<size_t>(s) * HDK_DEFL_MAX * jmax;
    for (int c = 0; c < kmin; ++c)
      for (int j = 0; j < m; ++j)
        cs[c * jmax + j] = Y[j * m + order[c]] * ((j & 1) ? -1.0 : 1.0) / std::sqrt(h[3 * j + 2]);
  }
  cuda_check(cudaMemcpyAsync(D.coef, D.h_coef, sizeof(double) * S * HDK_DEFL_MAX * jmax, cudaMemcpyHostToDevice, st_),
             "Ritz coefficients");
  hdk_check_p(hdk_sritz_combine(3 * dseg_.n, 3 * hf_.n, D.zhist, D.coef, jmax, kmin, D.w, st_), "Ritz vectors");
  D.k = kmin;
  D.valid = true;
  D.plain_iters = most;
  ++D.refreshes;
}

}  // namespace hdb
