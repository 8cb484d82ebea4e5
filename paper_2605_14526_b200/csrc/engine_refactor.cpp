// Engine::set_young on the device: after the first
// host build the pattern, the ordering, the elimination tree, the supernodes
// and the stream layout are fixed; a new material only changes values, so A
// is re-assembled, LDL^T re-factored (multifrontal) and S' rebuilt on the
// GPU, straight into the engine's buffers.  Reference: factor.cpp:11-136
// (SparseFactor::factorize, assemble_global_scalar), material.cpp set_young.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "engine.hpp"
#include "refactor.hpp"

namespace hdb {

namespace {
void hdk_check_r(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }
}  // namespace

struct Engine::DeviceRefactor {
  DevArena mem;
  hdk_mf mf{};
  std::vector<int> h_level_off, h_level_maxm;
  hdk_inverse_build build{};
  double *lx = nullptr, *d = nullptr, *dis = nullptr, *g = nullptr, *w = nullptr, *beta = nullptr;
  double* fd_tmp = nullptr;
  int *ff_off = nullptr, *ff_pair = nullptr, *ff_diag = nullptr, *fd_off = nullptr, *fd_pair = nullptr;
  int* df_from = nullptr;
  int* err = nullptr;
  int n_ff = 0, n_fd = 0;
};

void Engine::DeviceRefactorDeleter::operator()(DeviceRefactor* p) const { delete p; }

bool Engine::refactor_on_device() {
  if (const char* e = std::getenv("HETERODYN_HOST_REFACTOR"); e && std::atoi(e) != 0) return false;
  const HostFactor& F = hf_;
  if (!device_values_ || F.build.li.size() != F.build.lx.size() || F.build.parent.size() != static_cast<size_t>(F.n))
    return false;
  if (drf_) return true;
  auto R = std::unique_ptr<DeviceRefactor, DeviceRefactorDeleter>(new DeviceRefactor);
  DevArena& A = R->mem;
  const MfPlan P = mf_plan(F);
  const AssemblyPlan Q = assembly_plan(scene_.mesh, F);
  hdk_mf& v = R->mf;
  v.n = P.n;
  v.nsuper = P.nsuper;
  v.nlevels = P.nlevels;
  v.sfirst = A.upload(P.sfirst);
  v.fm = A.upload(P.fm);
  v.foff = A.upload(P.foff);
  v.level_off = A.upload(P.level_off);
  v.level_node = A.upload(P.level_node);
  v.child_off = A.upload(P.child_off);
  v.child = A.upload(P.child.empty() ? std::vector<int>{0} : P.child);
  v.emap_off = A.upload(P.emap_off);
  v.emap = A.upload(P.emap.empty() ? std::vector<int>{0} : P.emap);
  v.aent_off = A.upload(P.aent_off);
  v.aent_src = A.upload(P.aent_src);
  v.aent_dst = A.upload(P.aent_dst);
  v.lp = A.upload(P.lp);
  v.pool = A.alloc<double>(static_cast<size_t>(P.pool));
  R->h_level_off = P.level_off;
  v.h_level_off = R->h_level_off.data();
  R->h_level_maxm.assign(P.nlevels, 0);
  for (int L = 0; L < P.nlevels; ++L)
    for (int q = P.level_off[L]; q < P.level_off[L + 1]; ++q)
      R->h_level_maxm[L] = std::max(R->h_level_maxm[L], P.fm[P.level_node[q]]);
  v.h_level_maxm = R->h_level_maxm.data();
  R->lx = A.alloc<double>(static_cast<size_t>(P.lp[P.n]));
  R->d = A.alloc<double>(P.n);
  R->dis = A.alloc<double>(P.n);
  R->err = A.alloc<int>(1);
  // the S' builder's structural inputs stay resident; L and D^{-1/2} come from the fronts
  const DeviceBuild& B = F.build;
  hdk_inverse_build& b = R->build;
  b.n = F.n;
  b.max_depth = B.max_depth;
  b.tile_w = F.tile_w;
  b.parent = A.upload(B.parent);
  b.depth = A.upload(B.depth);
  b.lp = v.lp;
  b.ldist = A.upload(B.ldist.empty() ? std::vector<int>{0} : B.ldist);
  b.lx = R->lx;
  b.dis = R->dis;
  b.row_first = A.upload(B.row_first);
  b.row_pslot = A.upload(F.row_pslot);
  b.seg_off = A.upload(B.seg_off);
  b.seg_clo = A.upload(B.seg_clo);
  // assembly: shape gradients as factor.cpp assemble forms them
  const Mesh& m = scene_.mesh;
  Vec G(12 * static_cast<size_t>(m.ne));
  for (int e = 0; e < m.ne; ++e) {
    const double* bm = &m.bm[9 * static_cast<size_t>(e)];
    double* g = &G[12 * static_cast<size_t>(e)];
    for (int c = 0; c < 3; ++c) {
      g[3 + c] = bm[0 * 3 + c];
      g[6 + c] = bm[1 * 3 + c];
      g[9 + c] = bm[2 * 3 + c];
      g[c] = -(g[3 + c] + g[6 + c] + g[9 + c]);
    }
  }
  R->g = A.upload(G);
  R->w = A.alloc<double>(m.ne);
  R->beta = A.alloc<double>(m.ne);
  R->ff_off = A.upload(Q.ff_off);
  R->ff_pair = A.upload(Q.ff_pair.empty() ? std::vector<int>{0} : Q.ff_pair);
  R->ff_diag = A.upload(Q.ff_diag.empty() ? std::vector<int>{0} : Q.ff_diag);
  R->fd_off = A.upload(Q.fd_off);
  R->fd_pair = A.upload(Q.fd_pair.empty() ? std::vector<int>{0} : Q.fd_pair);
  R->df_from = A.upload(Q.df_from_fd.empty() ? std::vector<int>{0} : Q.df_from_fd);
  R->n_ff = static_cast<int>(Q.ff_diag.size());
  R->n_fd = static_cast<int>(Q.fd_off.size()) - 1;
  drf_ = std::move(R);
  return true;
}

// The numeric refactorization for mat_ (already updated and uploaded):
// assembly -> multifrontal LDL^T -> S' values, on st_.
void Engine::refactor_device_values() {
  DeviceRefactor& R = *drf_;
  const Mesh& m = scene_.mesh;
  const double h = scene_.solver.h;
  void* s = st_;
  // beta as upload_material staged it (pinned; set_young calls that first)
  cuda_check(cudaMemcpyAsync(R.beta, h_stage_ + 5 * static_cast<size_t>(m.ne), m.ne * sizeof(double),
                             cudaMemcpyHostToDevice, st_), "beta");
  cuda_check(cudaMemsetAsync(R.err, 0, sizeof(int), st_), "zero");
  hdk_check_r(hdk_asm_weights(m.ne, dmat_.mu_e, dmat_.lambda_e, R.beta, dmat_.vol, h, R.w, s), "A weights");
  const double inertia = (1.0 + mat_.alpha * h) / (h * h);
  hdk_check_r(hdk_asm_values(R.n_ff, R.ff_off, R.ff_pair, R.ff_diag, dm_.mass, inertia, R.w, R.g,
                             const_cast<double*>(a_ff_.val), s), "A_ff values");
  if (R.n_fd > 0) {
    hdk_check_r(hdk_asm_values(R.n_fd, R.fd_off, R.fd_pair, nullptr, dm_.mass, inertia, R.w, R.g,
                               const_cast<double*>(a_fd_.val), s), "A_fd values");
    hdk_check_r(hdk_gather_values(R.n_fd, R.df_from, a_fd_.val, const_cast<double*>(a_df_.val), s), "A_df values");
  }
  const bool trace = std::getenv("HETERODYN_REFACTOR_TRACE") != nullptr;
  cudaEvent_t ev[4] = {};
  if (trace)
    for (cudaEvent_t& e : ev) cuda_check(cudaEventCreate(&e), "event");
  if (trace) cuda_check(cudaEventRecord(ev[0], st_), "event");
  hdk_check_r(hdk_mf_factor(&R.mf, a_ff_.val, R.lx, R.d, R.dis, R.err, s), "multifrontal LDL^T");
  if (trace) cuda_check(cudaEventRecord(ev[1], st_), "event");
  hdk_check_r(hdk_inverse_values(&R.build, const_cast<double*>(df_.sval), s), "S' values");
  refresh_fp32();
  if (trace) {
    cuda_check(cudaEventRecord(ev[2], st_), "event");
    cuda_check(cudaEventSynchronize(ev[2]), "event");
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    std::fprintf(stderr, "[refactor] device: multifrontal LDL^T %.3f ms (%d levels, %d fronts), S' values %.3f ms\n", a,
                 R.mf.nlevels, R.mf.nsuper, b);
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  }
  int err = 0;
  cuda_check(cudaMemcpyAsync(&err, R.err, sizeof(int), cudaMemcpyDeviceToHost, st_), "refactor status");
  cuda_check(cudaStreamSynchronize(st_), "refactor");
  if (err) raise(Code::NotPositiveDefinite, "factor: non-positive pivot in the device refactorization");
  if (const char* v = std::getenv("HETERODYN_MF_VERIFY"); v && std::atoi(v) != 0) {
    // test hook: the device A values, L and D must equal the host assembly and
    // the CPU reference of the fronts (mf_factor_host) bit for bit
    const HostFactor H = build_factor(scene_.mesh, mat_, h, scene_.fixed, scene_.ordering, true, &order_cache_);
    Vec a(H.a_ff.val.size()), lx(H.build.lx.size()), d(H.n);
    cuda_check(cudaMemcpy(a.data(), a_ff_.val, a.size() * sizeof(double), cudaMemcpyDeviceToHost), "verify");
    cuda_check(cudaMemcpy(lx.data(), R.lx, lx.size() * sizeof(double), cudaMemcpyDeviceToHost), "verify");
    cuda_check(cudaMemcpy(d.data(), R.d, d.size() * sizeof(double), cudaMemcpyDeviceToHost), "verify");
    if (H.a_ff.val != a) raise(Code::InvalidArgument, "mf verify: device A values differ from the host assembly");
    const MfPlan P = mf_plan(hf_);
    Vec rlx, rd;
    mf_factor_host(P, H.a_ff.val, rlx, rd);
    if (rlx != lx || rd != d) raise(Code::InvalidArgument, "mf verify: device fronts differ from the CPU reference");
  }
}

}  // namespace hdb
