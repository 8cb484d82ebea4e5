// Device-resident forward/backward engine (see engine.hpp).
#include "engine.hpp"

#include <chrono>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>


namespace hdb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    raise(Code::InvalidArgument, std::string("CUDA failure in ") + what + ": " + cudaGetErrorString(e));
}
static void hdk_check(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

DevArena::~DevArena() {
  for (void* p : ptrs) cudaFree(p);
}
void cuda_zero(void* p, size_t bytes, const char* what) {
  cuda_check(cudaMemsetAsync(p, 0, bytes, cudaStreamLegacy), what);
  cuda_check(cudaStreamSynchronize(cudaStreamLegacy), what);
}

void* DevArena::raw(size_t bytes) {
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
  cuda_zero(p, bytes, "cudaMemset");
  ptrs.push_back(p);
  return p;
}
void DevArena::copy_h2d(void* d, const void* h, size_t bytes) { cuda_check(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice), "upload"); }

namespace {
cudaGraph_t capture(cudaStream_t st, const std::function<void()>& fn) {
  cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
  fn();
  cudaGraph_t g = nullptr;
  cuda_check(cudaStreamEndCapture(st, &g), "end capture");
  return g;
}
void capture_into(cudaStream_t st, cudaGraph_t body, const std::function<void()>& fn) {
  cuda_check(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
             "begin capture to graph");
  fn();
  cudaGraph_t out = nullptr;
  cuda_check(cudaStreamEndCapture(st, &out), "end capture to graph");
}
// pre -> while(body) -> post; returns the instantiated executable.  When
// conditional nodes are disabled the body is instantiated separately and the
// host drives the loop (debug fallback).
int kernel_nodes(cudaGraph_t g) {
  size_t n = 0;
  cuda_check(cudaGraphGetNodes(g, nullptr, &n), "graph nodes");
  std::vector<cudaGraphNode_t> nodes(n);
  if (n) cuda_check(cudaGraphGetNodes(g, nodes.data(), &n), "graph nodes");
  int k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    cuda_check(cudaGraphNodeGetType(nd, &t), "node type");
    if (t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

// pre -> while(body) -> post as one executable graph with a device-driven
// WHILE conditional node.  With conditional nodes disabled
// (HETERODYN_NO_COND_GRAPH=1, used for per-kernel profiling) pre, body and
// post are instantiated separately and the host drives the loop.
cudaGraphExec_t instantiate(cudaGraph_t g) {
  cudaGraphExec_t e = nullptr;
  cuda_check(cudaGraphInstantiate(&e, g, 0), "instantiate");
  return e;
}


cudaGraphExec_t capture_exec(cudaStream_t st, const std::function<void()>& fn, int* kernels) {
  cudaGraph_t g = capture(st, fn);
  if (kernels) *kernels = kernel_nodes(g);
  cudaGraphExec_t e = instantiate(g);
  cudaGraphDestroy(g);
  return e;
}
}  // namespace

void build_loop_graph(cudaStream_t st, bool use_cond, const std::function<void()>& pre,
                      const std::function<void(unsigned long long)>& body, const std::function<void()>& post,
                      LoopGraph& out) {
  out.destroy();
  cudaGraph_t gpre = capture(st, pre);
  cudaGraph_t gpost = capture(st, post);
  out.counts[0] = kernel_nodes(gpre);
  out.counts[2] = kernel_nodes(gpost);
  size_t npre_nodes = 0, npost_nodes = 0;
  cuda_check(cudaGraphGetNodes(gpre, nullptr, &npre_nodes), "graph nodes");
  cuda_check(cudaGraphGetNodes(gpost, nullptr, &npost_nodes), "graph nodes");
  if (!use_cond) {
    cudaGraph_t gbody = capture(st, [&] { body(0ULL); });
    out.counts[1] = kernel_nodes(gbody);
    out.pre = npre_nodes ? instantiate(gpre) : nullptr;
    out.body = instantiate(gbody);
    out.post = npost_nodes ? instantiate(gpost) : nullptr;
    for (cudaGraph_t g : {gpre, gbody, gpost}) cudaGraphDestroy(g);
    return;
  }
  cudaGraph_t top = nullptr;
  cuda_check(cudaGraphCreate(&top, 0), "graph create");
  cudaGraphNode_t npre, nloop, npost;
  const cudaGraphNode_t* dep = nullptr;
  size_t ndep = 0;
  if (npre_nodes) {
    cuda_check(cudaGraphAddChildGraphNode(&npre, top, nullptr, 0, gpre), "add pre");
    dep = &npre;
    ndep = 1;
  }
  cudaGraphConditionalHandle h;
  cuda_check(cudaGraphConditionalHandleCreate(&h, top, 1, cudaGraphCondAssignDefault), "cond handle");
  cudaGraphNodeParams p{};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cuda_check(cudaGraphAddNode(&nloop, top, dep, ndep, &p), "add while");
  capture_into(st, p.conditional.phGraph_out[0], [&] { body(static_cast<unsigned long long>(h)); });
  out.counts[1] = kernel_nodes(p.conditional.phGraph_out[0]);
  if (npost_nodes) cuda_check(cudaGraphAddChildGraphNode(&npost, top, &nloop, 1, gpost), "add post");
  out.exec = instantiate(top);
  for (cudaGraph_t g : {gpre, gpost, top}) cudaGraphDestroy(g);
}

void build_seq_graph(cudaStream_t st, bool use_cond, std::vector<SeqGraph::Seg> segs, SeqGraph& out) {
  out.destroy();
  const size_t ns = segs.size();
  out.kernels.assign(ns, 0);
  if (!use_cond) {
    out.parts.assign(ns, nullptr);
    for (size_t i = 0; i < ns; ++i) {
      cudaGraph_t g = capture(st, [&] { segs[i].fn(0ULL); });
      out.kernels[i] = kernel_nodes(g);
      out.parts[i] = instantiate(g);
      cudaGraphDestroy(g);
    }
  } else {
    cudaGraph_t top = nullptr;
    cuda_check(cudaGraphCreate(&top, 0), "graph create");
    std::vector<cudaGraphConditionalHandle> hs(ns, 0);
    for (size_t i = 0; i < ns; ++i)
      if (segs[i].loop)
        cuda_check(cudaGraphConditionalHandleCreate(&hs[i], top, segs[i].check_first ? 0 : 1, cudaGraphCondAssignDefault),
                   "cond handle");
    cudaGraphNode_t prev = nullptr;
    for (size_t i = 0; i < ns; ++i) {
      cudaGraphNode_t node = nullptr;
      if (!segs[i].loop) {
        const unsigned long long next = (i + 1 < ns && segs[i + 1].loop) ? static_cast<unsigned long long>(hs[i + 1]) : 0ULL;
        cudaGraph_t g = capture(st, [&] { segs[i].fn(next); });
        out.kernels[i] = kernel_nodes(g);
        size_t nn = 0;
        cuda_check(cudaGraphGetNodes(g, nullptr, &nn), "graph nodes");
        if (nn) {
          cuda_check(cudaGraphAddChildGraphNode(&node, top, prev ? &prev : nullptr, prev ? 1 : 0, g), "add segment");
          prev = node;
        }
        cudaGraphDestroy(g);
        continue;
      }
      cudaGraphNodeParams p{};
      p.type = cudaGraphNodeTypeConditional;
      p.conditional.handle = hs[i];
      p.conditional.type = cudaGraphCondTypeWhile;
      p.conditional.size = 1;
      cuda_check(cudaGraphAddNode(&node, top, prev ? &prev : nullptr, prev ? 1 : 0, &p), "add while");
      capture_into(st, p.conditional.phGraph_out[0], [&] { segs[i].fn(static_cast<unsigned long long>(hs[i])); });
      out.kernels[i] = kernel_nodes(p.conditional.phGraph_out[0]);
      prev = node;
    }
    out.exec = instantiate(top);
    cudaGraphDestroy(top);
  }
  for (auto& sg : segs) sg.fn = nullptr;  // captured; the closures may reference the caller's locals
  out.segs = std::move(segs);
}

Engine::Engine(const Scene& scene, const Vec* young, int solve_ctas, bool shared_device, int segments)
    : scene_(scene), mat_(scene.material), solve_ctas_(solve_ctas), branch_(!shared_device), segs_(segments) {
  if (segs_ < 1) raise(Code::InvalidArgument, "engine: segments must be >= 1");
  if (segs_ > 1) {
    if (!scene.obstacles.empty() || !scene.fixed.empty() || scene.hook || young)
      raise(Code::InvalidArgument, "segmented batch: contact-free scenes without Dirichlet vertices or hooks");
    if (scene.mesh.nv % segs_ || scene.mesh.ne % segs_ ||
        mat_.seg_means.size() != 3 * static_cast<size_t>(segs_))
      raise(Code::InvalidArgument, "segmented batch: the scene is not make_segmented_scene's");
  }
  if (const char* br = std::getenv("HETERODYN_BRANCH")) branch_ = std::atoi(br) != 0;
  if (const char* dv = std::getenv("HETERODYN_HOST_FACTOR_VALUES")) device_values_ = std::atoi(dv) == 0;
  if (const char* c = std::getenv("HETERODYN_SOLVE_CTAS")) solve_ctas_ = std::atoi(c);
  if (const char* u = std::getenv("HETERODYN_UNROLL")) unroll_ = std::max(1, std::atoi(u));
  if (young) mat_.set_young(*young, scene.mesh.vol);
  // adjoint backbone: preconditioned CG by default (same system and stopping
  // test as the reference's Anderson loop, half the iterations on C3);
  // HETERODYN_ADJOINT=aa keeps the reference's Anderson fixed point
  use_pcg_ = true;
  if (const char* ad = std::getenv("HETERODYN_ADJOINT")) use_pcg_ = std::string(ad) != "aa";
  {  // recycled-subspace deflation of the backbone CG (HETERODYN_DEFLATION=0: off; hd_sim_set_deflation).
     // Segmented (lockstep) engines: opt-in (=1) — C2-sized samples have few isolated slow modes
     // (40-41 vs 41-43 solves) and the per-sample (A - B)W costs more than it saves
    const char* e = std::getenv("HETERODYN_DEFLATION");
    defl_.on = segs_ > 1 ? (e && e[0] == '1') : !(e && e[0] == '0');
  }
  const char* nc = std::getenv("HETERODYN_NO_COND_GRAPH");
  use_cond_ = !(nc && std::atoi(nc) != 0);
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    raise(Code::InvalidArgument, "no CUDA device: the B200 engine has no CPU fallback");
  if (const char* ne = std::getenv("HETERODYN_NEWTON_EIGEN"))
    hdk_check(hdk_set_newton_eigen(std::atoi(ne) != 0 ? 1 : 0), "newton mode");
  cuda_check(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamCreateWithFlags(&st2_, cudaStreamNonBlocking), "stream");
  cuda_check(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming), "event");
  cuda_check(cudaMallocHost(&h_ctl_, sizeof(hdk_ctl) * segs_), "pinned ctl");
  if (const char* pe = std::getenv("HETERODYN_PHASES"); pe && std::atoi(pe) != 0) {
    ph_.on = true;
    ph_.per_frame = std::atoi(pe) == 2;
    for (cudaEvent_t& e : ph_.ev) cuda_check(cudaEventCreate(&e), "phase event");
  }
  fgraph_ = std::make_unique<LoopGraph>();
  bgraph_ = std::make_unique<LoopGraph>();
  eps_tr_ = scene.solver.eps_tr;
  if (segs_ > 1) {
    // the fill-reducing order of one copy, repeated per copy: the factor of
    // the block-diagonal operator is then block diagonal in sample order
    const int nvs = scene.mesh.nv / segs_, nes = scene.mesh.ne / segs_;
    Mesh m1;
    m1.nv = nvs;
    m1.ne = nes;
    m1.rest.assign(scene.mesh.rest.begin(), scene.mesh.rest.begin() + 3 * nvs);
    m1.el.assign(scene.mesh.el.begin(), scene.mesh.el.begin() + nes);
    m1.bm.assign(scene.mesh.bm.begin(), scene.mesh.bm.begin() + 9 * nes);
    m1.vol.assign(scene.mesh.vol.begin(), scene.mesh.vol.begin() + nes);
    m1.mass.assign(scene.mesh.mass.begin(), scene.mesh.mass.begin() + nvs);
    Material a1 = mat_;
    for (Vec* v : {&a1.young, &a1.mu, &a1.lambda, &a1.beta}) v->resize(nes);
    std::vector<int> ord1;
    build_factor(m1, a1, scene.solver.h, {}, scene.ordering, true, &ord1);
    order_cache_.resize(static_cast<size_t>(nvs) * segs_);
    for (int k = 0; k < segs_; ++k)
      for (int p = 0; p < nvs; ++p) order_cache_[static_cast<size_t>(k) * nvs + p] = k * nvs + ord1[p];
  }
  hf_ = build_factor(scene.mesh, mat_, scene.solver.h, scene.fixed, scene.ordering, device_values_, &order_cache_);
  refactor_count = 1;
  build_static();
  build_factor_device();
  build_forward_graph();
  build_backward_graph();
  time_ = 0;
}

void Engine::phase_mark(int i) {
  if (ph_.on) cuda_check(cudaEventRecord(ph_.ev[i], st_), "phase event");
}
// after a stream sync: accumulate the intervals between consecutive marks
void Engine::phase_collect(int first, int last) {
  if (!ph_.on) return;
  if (ph_.skip_first) {  // the first step also pays lazy module loading
    if (first == 0) ph_.skip_first = false;
    return;
  }
  for (int i = first; i < last; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ph_.ev[i], ph_.ev[i + 1]) == cudaSuccess) ph_.ms[i] += ms;
  }
  if (first == 0) ++ph_.n;
}

Engine::~Engine() {
  cols_.reset();
  if (ph_.on && ph_.n > 0) {
    static const char* names[7] = {"forward (graph + commit)", "-", "-", "backward pre", "backbone loop", "backward post",
                                   "-"};
    std::fprintf(stderr, "[heterodyn phases] %lld steps\n", ph_.n);
    for (int i : {0, 3, 4, 5}) std::fprintf(stderr, "  %-26s %9.3f ms/step\n", names[i], ph_.ms[i] / ph_.n);
    if (ph_.col_batches)
      std::fprintf(stderr, "  contact columns: %lld batches of %d, %.3f ms total, %lld batched iterations "
                   "(%.1f us each), %lld column iterations\n", ph_.col_batches, kColumns, ph_.col_ms,
                   ph_.col_iters, 1e3 * ph_.col_ms / std::max(1LL, ph_.col_iters), ph_.col_real_iters);
    std::fprintf(stderr, "  CG backbone fallbacks to Anderson (p.q <= 0): %lld; block-CG batches solved column by column: %lld\n",
                 pcg_fallbacks, bcg_fallbacks);
    std::fprintf(stderr, "  deflation: %lld recorded subspaces, %lld deflated solves (k = %d, recorded solve %d iterations)\n",
                 defl_.refreshes, defl_.deflated_solves, defl_.k, defl_.plain_iters);
  }
  for (cudaEvent_t e : ph_.ev)
    if (e) cudaEventDestroy(e);
  if (fgraph_) fgraph_->destroy();
  if (bgraph_) bgraph_->destroy();
  if (pgraph_) pgraph_->destroy();
  if (h_pcg_) cudaFreeHost(h_pcg_);
  cgraph_.destroy();
  for (cudaGraphExec_t e : {bpre_, bpost_a_, bpost_b_})
    if (e) cudaGraphExecDestroy(e);
  for (void* p : {static_cast<void*>(cM_), static_cast<void*>(cX_), static_cast<void*>(cz0_), ctr_mem_})
    if (p) cudaFree(p);
  if (h_cnt_) cudaFreeHost(h_cnt_);
  frame_mem_.clear();
  fmem_.reset();
  mem_.reset();
  if (h_ctl_) cudaFreeHost(h_ctl_);
  if (h_stage_) cudaFreeHost(h_stage_);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  if (st2_) cudaStreamDestroy(st2_);
  if (st_) cudaStreamDestroy(st_);
}

void Engine::build_static() {
  const Mesh& m = scene_.mesh;
  mem_ = std::make_unique<DevArena>();
  DevArena& A = *mem_;
  const size_t nv = m.nv, ne = m.ne, n3 = 3 * nv;
  std::vector<int> el(4 * ne);
  for (size_t e = 0; e < ne; ++e)
    for (int k = 0; k < 4; ++k) el[4 * e + k] = m.el[e][k];
  Vec bm(9 * ne);
  for (size_t e = 0; e < ne; ++e)
    for (int k = 0; k < 9; ++k) bm[k * ne + e] = m.bm[9 * e + k];
  // incidence lists in ascending element order (serial scatter order)
  std::vector<int> inc_off(nv + 1, 0), inc(4 * ne);
  for (size_t e = 0; e < ne; ++e)
    for (int k = 0; k < 4; ++k) ++inc_off[m.el[e][k] + 1];
  for (size_t v = 0; v < nv; ++v) inc_off[v + 1] += inc_off[v];
  {
    std::vector<int> cur(inc_off.begin(), inc_off.end() - 1);
    for (size_t e = 0; e < ne; ++e)
      for (int k = 0; k < 4; ++k) inc[cur[m.el[e][k]]++] = static_cast<int>(4 * e + k);
  }
  dm_.nv = m.nv;
  dm_.ne = m.ne;
  dm_.elem = A.upload(el);
  dm_.bm = A.upload(bm);
  dm_.mass = A.upload(m.mass);
  dm_.inc_off = A.upload(inc_off);
  dm_.inc = A.upload(inc);
  {  // corner -> its slot in the vertex-ordered incidence list (sorted forward forces)
    std::vector<int> cv(4 * ne);
    for (size_t j = 0; j < inc.size(); ++j) cv[inc[j]] = static_cast<int>(j);
    corner_vpos_ = A.upload(cv);
  }
  q_ = A.upload(scene_.q0);
  rest_ = A.upload(m.rest);
  v_ = A.upload(scene_.v0);
  fext_ = A.upload(external_force(scene_));
  qtil_ = A.alloc<double>(n3);
  qcur_ = A.alloc<double>(n3);
  qprev_ = A.alloc<double>(n3);
  qhat_ = A.alloc<double>(n3);
  bprev_ = A.alloc<double>(n3);
  damp_ = A.alloc<double>(n3);
  ef_ = A.alloc<double>(12 * ne);
  ef2_ = A.alloc<double>(12 * ne);
  lastq_ = A.alloc<double>(n3);
  lastg_ = A.alloc<double>(n3);
  dq_ = A.alloc<double>(HDK_AA_MAX * n3);
  dg_ = A.alloc<double>(HDK_AA_MAX * n3);
  part_a_ = A.alloc<double>(static_cast<size_t>(HDK_SEG_PSTRIDE) * segs_);
  part_b_ = A.alloc<double>(static_cast<size_t>(HDK_SEG_PSTRIDE) * segs_);
  part_c_ = A.alloc<double>(static_cast<size_t>(HDK_SEG_PSTRIDE) * segs_);
  cache_ = A.alloc<double>(24 * ne);
  ctl_ = A.alloc<hdk_ctl>(segs_);
  ticket_ = A.alloc<unsigned int>(segs_);
  snap_ = A.alloc<hdk_ctl>(segs_);
  if (segs_ > 1) {
    part18_ = A.alloc<double>(static_cast<size_t>(HDK_SEG_PSTRIDE) * segs_);
    cuda_zero(part18_, sizeof(double) * HDK_SEG_PSTRIDE * segs_, "zero partials");
    any_ = A.alloc<int>(1);
    gate_ticket_ = A.alloc<unsigned int>(1);
    cuda_zero(gate_ticket_, sizeof(unsigned int), "zero ticket");
    seg_windows_ = A.alloc<int>(2 * static_cast<size_t>(segs_));
    seg_means_dev_ = A.alloc<double>(3 * static_cast<size_t>(segs_));
  }
  dseg_.count = segs_;  // (a single problem is one segment for the hdk_seg_* loss / sum kernels)
  dseg_.nv = m.nv / segs_;
  dseg_.ne = m.ne / segs_;
  seed_ = A.alloc<double>(n3);
  x_ = A.alloc<double>(n3);
  t_ = A.alloc<double>(n3);
  bmu_ = A.alloc<double>(n3);
  dcomp_ = A.alloc<double>(30 * ne);
  qbar_ = A.alloc<double>(n3);
  vbar_ = A.alloc<double>(n3);
  dlq_ = A.alloc<double>(n3);
  dlv_ = A.alloc<double>(n3);
  dfacc_ = A.alloc<double>(n3);
  coup_ = A.alloc<double>(n3);
  dlw_ = A.alloc<double>(2 * ne);
  dle_ = A.alloc<double>(ne);
  eprev_ = A.alloc<double>(ne);
  estar_ = A.alloc<double>(ne);
  direct_ = A.alloc<double>(n3);
  bq_t_ = A.alloc<double>(n3);
  bv_t_ = A.alloc<double>(n3);
  bqtil_ = A.alloc<double>(n3);
  bqprev_ = A.alloc<double>(n3);
  bqstar_ = A.alloc<double>(n3);
  bcache_ = A.alloc<double>(24 * ne);
  mu_ = x_;
  dmat_.w1 = A.alloc<double>(ne);
  dmat_.w2 = A.alloc<double>(ne);
  dmat_.mu_e = A.alloc<double>(ne);
  dmat_.lambda_e = A.alloc<double>(ne);
  cuda_zero(ticket_, sizeof(unsigned int) * segs_, "zero tickets");
  dmat_.beta_vh = mat_.beta0 > 0 ? A.alloc<double>(ne) : nullptr;
  dmat_.vol = A.upload(m.vol);
  upload_material();
  const double hk[5] = {scene_.hook_anchor.x, scene_.hook_anchor.y, scene_.hook_anchor.z, scene_.hook_k, scene_.hook_d};
  hook_ = A.alloc<double>(5);
  DevArena::copy_h2d(hook_, hk, sizeof(hk));
  // obstacles: {kind, nx, ny, nz, offset|radius, cx, cy, cz, friction, 0, 0, 0}
  Vec ob;
  for (const Obstacle& o : scene_.obstacles) {
    const double rec[HDK_OBSTACLE_DOUBLES] = {static_cast<double>(o.kind), o.normal.x, o.normal.y, o.normal.z,
                                              o.kind == 0 ? o.offset : o.radius, o.center.x, o.center.y, o.center.z,
                                              o.friction, 0.0, 0.0, 0.0};
    ob.insert(ob.end(), rec, rec + HDK_OBSTACLE_DOUBLES);
  }
  obst_ = A.upload(ob);
  q0c_ = A.alloc<double>(n3);
  aa_window_ = scene_.solver.aa_window > 0 ? scene_.solver.aa_window : (mat_.contrast() > 10.0 ? 1 : 5);
  aa_window_ = std::min(aa_window_, HDK_AA_MAX);
}

// Material arrays (weights with volume folded in) and scalars into the
// existing device buffers; also the Anderson window, which follows the
// weight contrast (forward.cpp:56-83).
void Engine::upload_material() {
  const Mesh& m = scene_.mesh;
  const size_t ne = m.ne;
  const double h = scene_.solver.h;
  // pinned staging (w1, w2, mu, lambda, beta V / h, beta), filled by host
  // threads and copied asynchronously on st_ (a lockstep batch holds ~2 M
  // elements: pageable copies and one-thread loops cost ~30 ms per update)
  if (!h_stage_) cuda_check(cudaMallocHost(&h_stage_, 6 * ne * sizeof(double)), "pinned material stage");
  double *w1 = h_stage_, *w2 = w1 + ne, *mu = w2 + ne, *la = mu + ne, *bvh = la + ne, *beta = bvh + ne;
  const bool nh = mat_.kind == Kind::NeoHookean;
  parallel_ranges(static_cast<long long>(ne), [&](long long lo, long long hi) {
    for (long long e = lo; e < hi; ++e) {
      const double V = m.vol[e];
      if (nh) {
        w1[e] = mat_.weight(static_cast<int>(e)) * V;
        w2[e] = 0.0;
      } else {
        w1[e] = 2.0 * mat_.mu[e] * V;
        w2[e] = mat_.lambda[e] * V;
      }
      bvh[e] = mat_.beta[e] * V / h;
      mu[e] = mat_.mu[e];
      la[e] = mat_.lambda[e];
      beta[e] = mat_.beta[e];
    }
  }, 0, 1 << 15);
  dmat_.kind = nh ? 1 : 0;
  dmat_.barrier = mat_.barrier ? 1 : 0;
  dmat_.mu_bar = mat_.mu_bar;
  dmat_.lambda_bar = mat_.lambda_bar;
  dmat_.k_bar = mat_.k_bar;
  const auto put = [&](const double* d, const double* v) {
    cuda_check(cudaMemcpyAsync(const_cast<double*>(d), v, ne * sizeof(double), cudaMemcpyHostToDevice, st_),
               "upload material");
  };
  put(dmat_.w1, w1);
  put(dmat_.w2, w2);
  put(dmat_.mu_e, mu);
  put(dmat_.lambda_e, la);
  if (dmat_.beta_vh) put(dmat_.beta_vh, bvh);
  // weight range per sample (the whole mesh when not segmented): Anderson windows
  const int segs = segs_ > 1 ? segs_ : 1;
  const size_t sne = segs_ > 1 ? static_cast<size_t>(dseg_.ne) : ne;
  std::vector<double> lo(segs), hi(segs);
  parallel_ranges(segs, [&](long long k0, long long k1) {
    for (long long k = k0; k < k1; ++k) {
      double l = mat_.weight(static_cast<int>(k * sne)), u = l;
      for (size_t e = k * sne; e < (k + 1) * sne; ++e) {
        l = std::min(l, mat_.weight(static_cast<int>(e)));
        u = std::max(u, mat_.weight(static_cast<int>(e)));
      }
      lo[k] = l;
      hi[k] = u;
    }
  }, 0, 1);
  const double contrast = *std::max_element(hi.begin(), hi.end()) / *std::min_element(lo.begin(), lo.end());
  aa_window_ = scene_.solver.aa_window > 0 ? scene_.solver.aa_window : (contrast > 10.0 ? 1 : 5);
  aa_window_ = std::min(aa_window_, HDK_AA_MAX);
  if (segs_ > 1) {  // per-sample prox means and Anderson windows (each copy's own weight contrast)
    DevArena::copy_h2d(seg_means_dev_, mat_.seg_means.data(), mat_.seg_means.size() * sizeof(double));
    dmat_.seg_means = seg_means_dev_;
    dmat_.seg_ne = dseg_.ne;
    dmat_.tau_stride = static_cast<int>(sizeof(hdk_ctl) / sizeof(double));
    std::vector<int> win(2 * static_cast<size_t>(segs_), HDK_AA_MAX);
    for (int k = 0; k < segs_; ++k) {
      const int w = scene_.solver.aa_window > 0 ? scene_.solver.aa_window : (hi[k] / lo[k] > 10.0 ? 1 : 5);
      win[k] = std::min(w, HDK_AA_MAX);
    }
    DevArena::copy_h2d(seg_windows_, win.data(), win.size() * sizeof(int));
  }
  cuda_check(cudaStreamSynchronize(st_), "upload material");  // the stage is reused by the next update
}

// S' values of hf_ into the existing stream buffer (device build when the
// host left them to the device).
void Engine::fill_factor_values(double* sv) {
  const HostFactor& F = hf_;
  if (!F.stream.empty() || F.stream_len == 0) {
    DevArena::copy_h2d(sv, F.stream.data(), F.stream.size() * sizeof(double));
    return;
  }
  DevArena T;  // builder inputs, freed after the build
  const DeviceBuild& B = F.build;
  hdk_inverse_build b{};
  b.n = F.n;
  b.max_depth = B.max_depth;
  b.tile_w = F.tile_w;
  b.parent = T.upload(B.parent);
  b.depth = T.upload(B.depth);
  b.lp = T.upload(B.lp);
  b.ldist = T.upload(B.ldist.empty() ? std::vector<int>{0} : B.ldist);
  b.lx = T.upload(B.lx.empty() ? Vec{0.0} : B.lx);
  b.dis = T.upload(B.dis);
  b.row_first = T.upload(B.row_first);
  b.row_pslot = T.upload(F.row_pslot);
  b.seg_off = T.upload(B.seg_off);
  b.seg_clo = T.upload(B.seg_clo);
  hdk_check(hdk_inverse_values(&b, sv, st_), "device factor values");
  cuda_check(cudaStreamSynchronize(st_), "device factor values");
}

void Engine::refresh_fp32() {
  if (!df_.sval32) return;
  hdk_check(hdk_factor_to_fp32(&df_, const_cast<float*>(df_.sval32), df_.chunk32, st_), "fp32 factor values");
}

void Engine::build_factor_device() {
  fmem_ = std::make_unique<DevArena>();
  DevArena& A = *fmem_;
  const HostFactor& F = hf_;
  df_.n = F.n;
  df_.tile_w = F.tile_w;
  df_.n_tiles = static_cast<int>(F.tile_chunk.size()) - 1;
  df_.n_chunks = static_cast<int>(F.chunks.size());
  df_.max_ctas = 148 * 8;
  df_.grid_cap = solve_ctas_;
  {
    const char* hint = std::getenv("HETERODYN_L2_HINT");
    df_.l2_hint = hint ? std::atoi(hint) : 1;
  }
  {
    double* sv = A.alloc<double>(static_cast<size_t>(std::max<long long>(F.stream_len, F.stream.size())));
    fill_factor_values(sv);
    df_.sval = sv;
  }
  static_assert(sizeof(hdk_seg) == sizeof(SegDesc), "segment descriptor layout");
  static_assert(sizeof(hdk_chunk) == sizeof(ChunkDesc), "chunk descriptor layout");
  hdk_seg* segs = A.alloc<hdk_seg>(F.sdesc.size());
  DevArena::copy_h2d(segs, F.sdesc.data(), sizeof(SegDesc) * F.sdesc.size());
  df_.seg = segs;
  hdk_chunk* ch = A.alloc<hdk_chunk>(F.chunks.size());
  DevArena::copy_h2d(ch, F.chunks.data(), sizeof(ChunkDesc) * F.chunks.size());
  df_.chunk = ch;
  if (const char* e32 = std::getenv("HETERODYN_PCG_FP32"); e32 && e32[0] == '1') {
    // fp32 copy of the stream for the adjoint CG's preconditioner solves
    // (opt-in, engine_pcg.cpp); chunks padded to 4 values
    std::vector<ChunkDesc> c32(F.chunks.begin(), F.chunks.end());
    long long off = 0;
    for (ChunkDesc& c : c32) {
      c.off = off;
      c.len = (c.len + 3) & ~3;
      off += c.len;
    }
    hdk_chunk* ch32 = A.alloc<hdk_chunk>(c32.size());
    DevArena::copy_h2d(ch32, c32.data(), sizeof(ChunkDesc) * c32.size());
    df_.chunk32 = ch32;
    df_.sval32 = A.alloc<float>(static_cast<size_t>(std::max(off, 4LL)));
    df_.use32 = 0;  // exact solves by default; the CG's factor view sets it
    refresh_fp32();
  }
  df_.tile_chunk = A.upload(F.tile_chunk);
  df_.row_pslot = A.upload(F.row_pslot);
  df_.n_pslot = F.row_pslot.back();
  {  // z-fold warp tasks (solve.cu zfold_task)
    std::vector<int> zt;
    for (int r = 0; r < F.n;) {
      if (F.row_pslot[r + 1] - F.row_pslot[r] > 8) {
        zt.push_back(r);
        zt.push_back(-1);
        ++r;
        continue;
      }
      int k = 0;
      while (k < 4 && r + k < F.n && F.row_pslot[r + k + 1] - F.row_pslot[r + k] <= 8) ++k;
      zt.push_back(r);
      zt.push_back(k);
      r += k;
    }
    df_.n_ztask = static_cast<int>(zt.size() / 2);
    df_.ztask = reinterpret_cast<const int2*>(A.upload(zt));
  }
  df_.p2v = A.upload(F.p2v);
  df_.v2p = A.upload(F.v2p);
  df_.part1 = A.alloc<double>(3 * static_cast<size_t>(F.row_pslot.back()));
  df_.part2 = A.alloc<double>(3 * static_cast<size_t>(F.tile_w) * (df_.n_tiles + df_.max_ctas));
  df_.z = A.alloc<double>(3 * static_cast<size_t>(F.n));
  // cost-balanced CTA ranges for the grids the solve will launch: a segment
  // costs about as much as 300 (pass 1) / 200 (pass 2) streamed values
  // (per-CTA traces of the C3 factor, scripts/micro/solve_bench.cu)
  {
    int g1 = 0, g2 = 0;
    hdk_check(hdk_solve_grids(&df_, &g1, &g2), "solve grids");
    const auto env_cost = [](const char* name, double dflt) {
      const char* v = std::getenv(name);
      return v ? std::atof(v) : dflt;
    };
    const std::vector<int> f1 = balanced_ranges(F.chunks, g1, env_cost("HETERODYN_SEG_COST1", 300.0));
    const std::vector<int> f2 = balanced_ranges(F.chunks, g2, env_cost("HETERODYN_SEG_COST2", 200.0));
    df_.grid1 = g1;
    df_.grid2 = g2;
    df_.first1 = A.upload(f1);
    df_.first2 = A.upload(f2);
    const std::vector<int> tc = tile_cta_ranges(F.tile_chunk, f2);
    df_.tile_cta2 = A.upload(tc);
    // per vertex: first pass-2 tile-partial slot of its column and how many
    // CTAs wrote one (0 for fixed vertices) — the x-fold's one indirection
    std::vector<int> vf(2 * static_cast<size_t>(scene_.mesh.nv), 0);
    for (int c = 0; c < F.n; ++c) {
      const int t = c / F.tile_w, v = F.p2v[c];
      vf[2 * v] = (t + tc[2 * t]) * F.tile_w + (c - t * F.tile_w);
      vf[2 * v + 1] = tc[2 * t + 1] - tc[2 * t] + 1;
    }
    df_.vfold = reinterpret_cast<const int2*>(A.upload(vf));

  }
  rhs_ = A.alloc<double>(3 * static_cast<size_t>(F.n));
  fixc_ = A.alloc<double>(3 * static_cast<size_t>(F.n));
  dqp_ = A.alloc<double>(3 * static_cast<size_t>(F.n));
  auto up_csr = [&](const Csr& c, hdk_csr& d) {
    d.rows = c.rows;
    d.off = A.upload(c.off);
    d.col = A.upload(c.col);
    d.val = A.upload(c.val);
  };
  up_csr(F.a_ff, a_ff_);
  up_csr(F.a_fd, a_fd_);
  // A_df = A_fd^T (fixed rows x free columns)
  Csr t;
  t.rows = F.a_fd.cols;
  t.cols = F.n;
  t.off.assign(t.rows + 1, 0);
  for (int c : F.a_fd.col) ++t.off[c + 1];
  for (int r = 0; r < t.rows; ++r) t.off[r + 1] += t.off[r];
  t.col.resize(F.a_fd.col.size());
  t.val.resize(F.a_fd.col.size());
  {
    std::vector<int> cur(t.off.begin(), t.off.end() - 1);
    for (int p = 0; p < F.a_fd.rows; ++p)
      for (int k = F.a_fd.off[p]; k < F.a_fd.off[p + 1]; ++k) {
        const int pos = cur[F.a_fd.col[k]]++;
        t.col[pos] = p;
        t.val[pos] = F.a_fd.val[k];
      }
  }
  up_csr(t, a_df_);
  d_fixed_ = A.upload(F.fixed.empty() ? std::vector<int>{0} : F.fixed);
  dv_.nv = scene_.mesh.nv;
  dv_.n = F.n;
  dv_.v2p = df_.v2p;
  dv_.p2v = df_.p2v;
  dv_.mass = dm_.mass;
  dv_.inc_off = dm_.inc_off;
  dv_.inc = dm_.inc;
  {  // incidence lists in elimination order (same per-vertex order)
    const Mesh& m = scene_.mesh;
    std::vector<int> cnt(m.nv, 0);
    for (size_t e = 0; e < m.ne; ++e)
      for (int k = 0; k < 4; ++k) ++cnt[m.el[e][k]];
    std::vector<int> voff(m.nv + 1, 0);
    for (int v = 0; v < m.nv; ++v) voff[v + 1] = voff[v] + cnt[v];
    std::vector<int> vinc(voff[m.nv]);
    {
      std::vector<int> cur(voff.begin(), voff.end() - 1);
      for (size_t e = 0; e < m.ne; ++e)
        for (int k = 0; k < 4; ++k) vinc[cur[m.el[e][k]]++] = static_cast<int>(4 * e + k);
    }
    std::vector<int> poff(F.n + 1, 0), pinc;
    pinc.reserve(vinc.size());
    for (int p = 0; p < F.n; ++p) {
      const int v = F.p2v[p];
      pinc.insert(pinc.end(), vinc.begin() + voff[v], vinc.begin() + voff[v + 1]);
      poff[p + 1] = static_cast<int>(pinc.size());
    }
    dv_.pinc_off = A.upload(poff);
    dv_.pinc = A.upload(pinc.empty() ? std::vector<int>{0} : pinc);
    // corner -> its slot in pinc (hdk_bapply_sorted); -1 for fixed vertices
    std::vector<int> cpos(4 * static_cast<size_t>(m.ne), -1);
    for (size_t j = 0; j < pinc.size(); ++j) cpos[pinc[j]] = static_cast<int>(j);
    corner_pos_ = A.upload(cpos);
  }
  seedp_ = A.alloc<double>(3 * static_cast<size_t>(F.n));
  xp_ = A.alloc<double>(3 * static_cast<size_t>(F.n));
  dseg_.n = F.n / segs_;
  if (segs_ > 1) {  // the postordered elimination order must keep every sample's block contiguous
    const int ns = F.n / segs_, nvs = scene_.mesh.nv / segs_;
    bool ok = F.n % segs_ == 0;
    for (int p = 0; ok && p < F.n; ++p) ok = F.p2v[p] / nvs == p / ns;
    if (!ok) raise(Code::InvalidArgument, "segmented batch: elimination order mixes samples");
    dseg_.n = ns;
  }
  {
    const size_t n3p = 3 * static_cast<size_t>(F.n);
    rt_ = A.alloc<double>(n3p);
    rx_ = A.alloc<double>(n3p);
    lrx_ = A.alloc<double>(n3p);
    lrg_ = A.alloc<double>(n3p);
    rsq_ = A.alloc<double>(HDK_AA_MAX * n3p);
    tv_ = A.alloc<double>(3 * static_cast<size_t>(scene_.mesh.nv));
    aares_ = A.raw(hdk_bb_result_bytes() * segs_);
  }
}

void Engine::build_forward_graph() {
  if (segs_ > 1) {
    build_forward_graph_seg();
    return;
  }
  const Solver& so = scene_.solver;
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  const double h = so.h;
  const double hk[5] = {scene_.hook_anchor.x, scene_.hook_anchor.y, scene_.hook_anchor.z, scene_.hook_k, scene_.hook_d};
  void* s = st_;
  auto pre = [&] {
    hdk_check(hdk_ctl_init(ctl_, aa_window_, 10.0, so.k_max, so.eps_rel, so.eps_abs, 0.0, so.eps_tr, 0, s), "ctl init");
    hdk_check(hdk_free_fall(&dv_, q_, v_, fext_, h, scene_.hook ? scene_.hook_vertex : -1, scene_.hook ? hk : nullptr,
                            qtil_, qcur_, s), "free fall");
    if (dmat_.beta_vh) hdk_check(hdk_damping_elements(&dm_, dmat_.beta_vh, q_, ef2_, s), "damping elements");
    hdk_check(hdk_gather(&dv_, dmat_.beta_vh ? ef2_ : nullptr, mat_.alpha / h, q_, nullptr, damp_, s), "damping gather");
    if (!hf_.fixed.empty()) hdk_check(hdk_fixed_coupling(&a_fd_, d_fixed_, q_, fixc_, s), "fixed coupling");
    cuda_check(cudaMemcpyAsync(qhat_, q_, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st_), "qhat init");
  };
  auto body = [&](unsigned long long handle) {
    hdk_check(hdk_local_step_sorted(&dm_, &dmat_, qcur_, ef_, &ctl_->err, corner_vpos_, s), "local step");
    hdk_check(hdk_gather_rhs_sorted(&dv_, ef_, 1.0 / (h * h), qtil_, damp_, hf_.fixed.empty() ? nullptr : fixc_, bprev_, rhs_,
                             part_a_, s), "rhs");
    hdk_check(hdk_apply_inverse3_partial(&df_, rhs_, s), "solve");
    hdk_check(hdk_aa_dots_fused(&dv_, &df_, ctl_, qhat_, qcur_, lastq_, lastg_, dq_, dg_, part_b_, ticket_, 0, 0ULL, s),
              "aa dots + solve");
    hdk_check(hdk_aa_mix(&dv_, ctl_, qhat_, qcur_, qprev_, q_, dq_, dg_, part_c_, 0, s), "aa mix");
    hdk_check(hdk_gate(ctl_, part_a_, part_c_, handle, s), "gate");
  };
  auto post = [&] {
    hdk_check(hdk_local_step(&dm_, &dmat_, qcur_, ef_, cache_, &ctl_->err, s), "cache sweep");
  };
  build_loop_graph(st_, use_cond_, pre, body, post, *fgraph_);
  if (cw_.base) build_contact_graph();  // scenes with obstacles (engine_contact.cpp)
  fk_pre_ = fgraph_->counts[0];
  fk_body_ = fgraph_->counts[1];
  fk_post_ = fgraph_->counts[2];
}

void Engine::build_backward_graph() {
  if (pgraph_) pgraph_->destroy();  // rebuilt on first use (it bakes factor and material pointers)
  pgraph_.reset();
  if (segs_ > 1) {
    build_backward_graph_seg();
    return;
  }
  const Solver& so = scene_.solver;
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  const double h = so.h;
  const bool has_fixed = !hf_.fixed.empty();
  const double umu = 1.0 / (2.0 * (1.0 + mat_.poisson));  // lame(1, nu) (backward.cpp:363)
  const double ula = mat_.poisson / ((1.0 + mat_.poisson) * (1.0 - 2.0 * mat_.poisson));
  void* s = st_;
  for (cudaGraphExec_t* e : {&bpre_, &bpost_a_, &bpost_b_})
    if (*e) {
      cudaGraphExecDestroy(*e);
      *e = nullptr;
    }
  // tr_select_tau, differential, seed and the backbone's first solve
  bpre_ = capture_exec(st_, [&] {
    hdk_check(hdk_ctl_init(ctl_, HDK_AA_MAX, 1e8, 500, 0.0, 0.0, 1e-10, eps_tr_, 0, s), "ctl init");
    hdk_check(hdk_tr_model(&dv_, &a_ff_, bqstar_, bqprev_, dqp_, part_a_, s), "tr model");
    hdk_check(hdk_element_energy2(&dm_, &dmat_, bqprev_, eprev_, bqstar_, estar_, &ctl_->bad, s), "energies");
    hdk_check(hdk_tr_select(&dv_, dm_.ne, eprev_, estar_, bqprev_, bqstar_, bqtil_, 1.0 / (h * h), part_a_, part_b_,
                            ctl_, s), "tr select");
    hdk_check(hdk_differential(&dm_, &dmat_, bcache_, &ctl_->tau, dcomp_, &ctl_->err, s), "differential");
    hdk_check(hdk_axpby(static_cast<int>(n3), 1.0, qbar_, 1.0 / h, vbar_, seed_, s), "seed");
    cuda_check(cudaMemsetAsync(x_, 0, n3 * sizeof(double), st_), "x zero");
    cuda_check(cudaMemsetAsync(t_, 0, n3 * sizeof(double), st_), "t zero");
    hdk_check(hdk_gather_perm(&dv_, seed_, nullptr, rhs_, s), "x0 rhs");
    hdk_check(hdk_apply_inverse3(&df_, rhs_, x_, s), "x0 solve");
  }, &bk_pre_);
  // backbone fixed point x <- A^{-1}(seed + B x) with AA(8) (backward.cpp:170-204);
  // the loop's pre step forms the first right-hand side seed + R(x0), R = gather o B
  // (also run for each contact column, which re-seeds seed_ and x_)
  auto pre = [&] {
    hdk_check(hdk_aa_reset(ctl_, HDK_AA_MAX, 1e8, 500, 1e-10, s), "aa reset");
    hdk_check(hdk_gather_perm(&dv_, seed_, nullptr, seedp_, s), "seed in elimination order");
    hdk_check(hdk_gather_perm(&dv_, x_, nullptr, xp_, s), "x0 in elimination order");
    hdk_check(hdk_bapply(&dm_, dcomp_, x_, ef_, s), "B x0");
    hdk_check(hdk_gather_pp(&dv_, nullptr, ef_, rx_, nullptr, s), "R(x0)");
    hdk_check(hdk_axpby(3 * hf_.n, 1.0, seedp_, 1.0, rx_, rhs_, s), "rhs0");
  };
  auto body = [&](unsigned long long handle) {
    for (int u = 0; u < unroll_; ++u) {
      if (loop_trace_) hdk_check(hdk_trace_epoch(loop_trace_, s), "trace epoch");
      backbone_body(handle, 0u);
    }
  };
  build_loop_graph(st_, use_cond_, pre, body, [] {}, *bgraph_);
  bk_body_ = bgraph_->counts[1];
  bk_pre_ += bgraph_->counts[0];
  // gradient routing (backward.cpp:286-394); the contact path adds the
  // friction pushback between the two halves
  bpost_a_ = capture_exec(st_, [&] {
    if (has_fixed) {
      hdk_check(hdk_bapply(&dm_, dcomp_, x_, ef_, s), "B mu");
      hdk_check(hdk_gather(&dv_, ef_, 0.0, x_, nullptr, bmu_, s), "B mu gather");
      hdk_check(hdk_fixed_coupling_t(&a_df_, d_fixed_, df_.p2v, x_, coup_, s), "A_fd^T mu");
    }
    hdk_check(hdk_route_elements(&dm_, &dmat_, bcache_, bqstar_, x_, umu, ula, dlw_, dle_,
                                 dmat_.beta_vh ? ef2_ : nullptr, s), "route elements");
    hdk_check(hdk_route_vertices(&dv_, x_, dmat_.beta_vh ? ef2_ : nullptr, has_fixed ? bmu_ : nullptr, qbar_, vbar_,
                                 has_fixed ? coup_ : nullptr, h, mat_.alpha, scene_.hook ? scene_.hook_vertex : -1,
                                 scene_.hook_k, scene_.hook_d, dlq_, dlv_, dfacc_, s), "route vertices");
  }, &bk_post_);
  int kb = 0;
  bpost_b_ = capture_exec(st_, [&] {
    hdk_check(hdk_axpby(static_cast<int>(n3), 1.0, dlq_, 1.0, direct_, qbar_, s), "next q seed");
    hdk_check(hdk_axpby(static_cast<int>(n3), 1.0, dlv_, 0.0, nullptr, vbar_, s), "next v seed");
  }, &kb);
  bk_post_ += kb;
}

// One adjoint backbone iteration x <- A^{-1}(seed + B x) + AA(8)
// (backward.cpp:170-204); skip bits drop kernels for timing ablations only.
// The loop graph holds unroll_ copies of it; every kernel of a copy past
// convergence returns at once (ctl->cond == 0), so one WHILE re-launch covers
// unroll_ iterations.
//   solve(rhs) -> dots(t) -> { coefficient solve || R(t) = gather(B t) } -> mix,
// the coefficient solve on a second branch of the graph (st2_).
void Engine::backbone_body(unsigned long long handle, unsigned skip) {
  void* s = st_;
  hdk_factor fb = df_;
  fb.run_flag = &ctl_->cond;
  const int* run_it = &snap_->cond;  // fixed for the iteration (ctl->cond moves with the branch's solve)
  if (!(skip & 4u)) hdk_check(hdk_apply_inverse3_ablate(&fb, rhs_, (skip >> 6) & 7u, s), "solve");
  if (!(skip & 8u))
    hdk_check(hdk_bb_dots(&df_, ctl_, snap_, t_, tv_, xp_, lastq_, lastg_, dq_, dg_, part_b_, 1 | (skip & (512u | 1024u)),
                          s),
              "aa dots");
  // a batch's engines keep one stream each (the device is already shared by
  // many samples, and every extra stream competes for the hardware queues)
  cudaStream_t sb = branch_ ? st2_ : st_;
  if (branch_) {
    cuda_check(cudaEventRecord(ev_fork_, st_), "fork");
    cuda_check(cudaStreamWaitEvent(st2_, ev_fork_, 0), "fork wait");
  }
  if (!(skip & 16u)) hdk_check(hdk_bb_solve(ctl_, snap_, part_b_, aares_, handle, sb), "aa solve + cond");
  if (!(skip & 1u)) hdk_check(hdk_bapply_sorted(&dm_, dcomp_, tv_, ef_, corner_pos_, run_it, s), "B t");
  if (!(skip & 2u)) hdk_check(hdk_gather_sorted(&dv_, nullptr, ef_, rt_, run_it, s), "R(t)");
  if (branch_) {
    cuda_check(cudaEventRecord(ev_join_, st2_), "join");
    cuda_check(cudaStreamWaitEvent(st_, ev_join_, 0), "join wait");
  }
  if (!(skip & 16u))
    hdk_check(hdk_bb_mix(&df_, ctl_, snap_, aares_, t_, xp_, x_, dq_, rt_, rx_, lrx_, lrg_, rsq_, seedp_, rhs_, s),
              "aa mix");
}

double Engine::time_backbone(int reps, unsigned skip) {
  if (std::getenv("HETERODYN_BODY_DIRECT")) {  // plain stream launches (ncu cannot profile graph
    for (int i = 0; i < reps; ++i) backbone_body(0ULL, skip);  // nodes that may set a condition)
    cuda_check(cudaStreamSynchronize(st_), "direct body");
    return 0.0;
  }
  cudaGraphExec_t g = capture_exec(st_, [&] { backbone_body(0ULL, skip); }, nullptr);
  cudaEvent_t a, b;
  cuda_check(cudaEventCreate(&a), "event");
  cuda_check(cudaEventCreate(&b), "event");
  for (int i = 0; i < 3; ++i) cuda_check(cudaGraphLaunch(g, st_), "warm body");
  cuda_check(cudaEventRecord(a, st_), "event");
  for (int i = 0; i < reps; ++i) cuda_check(cudaGraphLaunch(g, st_), "timed body");
  cuda_check(cudaEventRecord(b, st_), "event");
  cuda_check(cudaEventSynchronize(b), "event sync");
  float ms = 0;
  cuda_check(cudaEventElapsedTime(&ms, a, b), "elapsed");
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaGraphExecDestroy(g);
  return static_cast<double>(ms) / reps;
}

// Timeline of `reps` consecutive backbone iterations (profiling): per
// iteration and kernel {first CTA resident, first CTA past its PDL wait, last
// CTA end} in ns; out holds reps x kTrCount x 3 values relative to the first.
void Engine::trace_backbone(int reps, std::vector<double>& out) {
  constexpr int kSlots = 16, kK = 14;
  reps = std::max(1, std::min(reps, kSlots));
  const size_t words = 1 + 3 * static_cast<size_t>(kSlots) * kK;
  unsigned long long* buf = nullptr;
  cuda_check(cudaMalloc(&buf, words * 8), "trace buffer");
  std::vector<unsigned long long> h(words);
  for (size_t i = 1; i < words; i += 3) {
    h[i] = ~0ULL;
    h[i + 1] = ~0ULL;
    h[i + 2] = 0ULL;
  }
  h[0] = kSlots - 1;  // first epoch bump lands on slot 0
  cuda_check(cudaMemcpy(buf, h.data(), words * 8, cudaMemcpyHostToDevice), "trace init");
  for (auto inst : {hdk_trace_install_local, hdk_trace_install_vec, hdk_trace_install_solve})
    hdk_check(inst(buf), "trace install");
  cudaGraphExec_t g = capture_exec(st_, [&] {
    hdk_check(hdk_trace_epoch(buf, st_), "trace epoch");
    const char* sk = std::getenv("HETERODYN_TRACE_SKIP");
    backbone_body(0ULL, sk ? static_cast<unsigned>(std::atoi(sk)) : 0u);
  }, nullptr);
  for (int i = 0; i < reps; ++i) cuda_check(cudaGraphLaunch(g, st_), "traced body");
  cuda_check(cudaStreamSynchronize(st_), "trace sync");
  cudaGraphExecDestroy(g);
  for (auto inst : {hdk_trace_install_local, hdk_trace_install_vec, hdk_trace_install_solve})
    hdk_check(inst(nullptr), "trace uninstall");
  cuda_check(cudaMemcpy(h.data(), buf, words * 8, cudaMemcpyDeviceToHost), "trace read");
  cudaFree(buf);
  unsigned long long t0 = ~0ULL;
  for (int r = 0; r < reps; ++r)
    for (int k = 0; k < kK; ++k) t0 = std::min(t0, h[1 + 3 * (r * kK + k)]);
  out.assign(static_cast<size_t>(reps) * kK * 3, -1.0);
  for (int r = 0; r < reps; ++r)
    for (int k = 0; k < kK; ++k)
      for (int j = 0; j < 3; ++j) {
        const unsigned long long v = h[1 + 3 * (r * kK + k) + j];
        if (v != ~0ULL && v != 0ULL) out[3 * (r * kK + k) + j] = static_cast<double>(v - t0);
      }
}

// Timeline of the real backbone WHILE loop (profiling): one recorded
// forward step from the current state, then its backward with an epoch
// kernel in front of every unrolled iteration; out receives the last
// min(iterations, 16) iterations' records (same layout as trace_backbone,
// oldest first).  The state is restored afterwards.
void Engine::trace_loop(std::vector<double>& out) {
  constexpr int kSlots = 16, kK = 14;
  const size_t words = 1 + 3 * static_cast<size_t>(kSlots) * kK;
  std::vector<unsigned long long> h(words);
  for (size_t i = 1; i < words; i += 3) {
    h[i] = ~0ULL;
    h[i + 1] = ~0ULL;
    h[i + 2] = 0ULL;
  }
  h[0] = kSlots - 1;
  cuda_check(cudaMalloc(&loop_trace_, words * 8), "trace buffer");
  cuda_check(cudaMemcpy(loop_trace_, h.data(), words * 8, cudaMemcpyHostToDevice), "trace init");
  build_backward_graph();
  const Vec q = positions(), v = velocities();
  const double t = time_;
  record(true);
  step();
  for (auto inst : {hdk_trace_install_local, hdk_trace_install_vec, hdk_trace_install_solve})
    hdk_check(inst(loop_trace_), "trace install");
  backward(nullptr, nullptr, nullptr, true, false, nullptr);
  cuda_check(cudaStreamSynchronize(st_), "trace sync");
  for (auto inst : {hdk_trace_install_local, hdk_trace_install_vec, hdk_trace_install_solve})
    hdk_check(inst(nullptr), "trace uninstall");
  cuda_check(cudaMemcpy(h.data(), loop_trace_, words * 8, cudaMemcpyDeviceToHost), "trace read");
  cudaFree(loop_trace_);
  loop_trace_ = nullptr;
  build_backward_graph();
  record(false);
  set_state(q.data(), v.data(), t);
  const int iters = last_backward_iterations_;
  const int nrec = std::min(iters, kSlots);
  const unsigned long long ep = h[0];  // slot of the last epoch
  unsigned long long t0 = ~0ULL;
  for (int k = 0; k < nrec; ++k) {
    const int slot = static_cast<int>((ep + kSlots - (nrec - 1 - k)) % kSlots);
    for (int j = 0; j < kK; ++j) t0 = std::min(t0, h[1 + 3 * (slot * kK + j)]);
  }
  out.assign(static_cast<size_t>(nrec) * kK * 3, -1.0);
  for (int k = 0; k < nrec; ++k) {
    const int slot = static_cast<int>((ep + kSlots - (nrec - 1 - k)) % kSlots);
    for (int j = 0; j < kK; ++j)
      for (int c = 0; c < 3; ++c) {
        const unsigned long long val = h[1 + 3 * (slot * kK + j) + c];
        if (val != ~0ULL && val != 0ULL) out[3 * (k * kK + j) + c] = static_cast<double>(val - t0);
      }
  }
}

void Engine::sync_ctl() {
  cuda_check(cudaMemcpyAsync(h_ctl_, ctl_, sizeof(hdk_ctl) * segs_, cudaMemcpyDeviceToHost, st_), "ctl read");
  cuda_check(cudaStreamSynchronize(st_), "stream sync");
}

void Engine::run_graph(LoopGraph& g, const char* what) {
  if (g.exec) {
    cuda_check(cudaGraphLaunch(g.exec, st_), what);
    return;
  }
  // host-driven loop (profiling fallback): one status read per iteration
  if (g.pre) cuda_check(cudaGraphLaunch(g.pre, st_), what);
  for (;;) {
    cuda_check(cudaGraphLaunch(g.body, st_), what);
    sync_ctl();
    if (segs_ > 1 ? !host_any() : !h_ctl_->cond) break;
  }
  if (g.post) cuda_check(cudaGraphLaunch(g.post, st_), what);
}

void Engine::check_ctl(const char* what) {
  for (int k = 0; k < segs_; ++k) {
    hdk_ctl* hc = h_ctl_ + k;
    if (hc->err == 0 && hc->nonfinite) hc->err = 10;  // non-finite backbone iterate
    if (hc->err == 0) continue;
    const int c = hc->err;
    std::string msg = std::string(what) + (segs_ > 1 ? " (sample " + std::to_string(k) + ")" : std::string()) + ": ";
    switch (c) {
      case 6: msg += "local stretch solve did not reach stationarity"; break;
      case 7: msg += "filtered prox Hessian is numerically singular"; break;
      case 9: msg += "contact system is singular even after the diagonal lift"; break;
      case 10: msg += "adjoint backbone iteration did not settle (cap or non-finite values)"; break;
      default: msg += "device solver error"; break;
    }
    raise(static_cast<Code>(c), msg);
  }
}

void Engine::step() {
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv), ne = scene_.mesh.ne;
  const bool contact_scene = !scene_.obstacles.empty();
  phase_mark(0);
  if (contact_scene) run_contact_step();
  else run_graph(*fgraph_, "forward graph");
  const bool rec = recording_ || force_slot_ >= 0;
  const int slot = force_slot_ >= 0 ? force_slot_ : nrec_;
  if (rec) {
    while (static_cast<int>(slots_.size()) <= slot) add_slot();
    const Frame& fr = slots_[slot];
    const auto cp = [&](double* d, const double* src, size_t n) {
      cuda_check(cudaMemcpyAsync(d, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st_), "record");
    };
    cp(fr.q_t, q_, n3);
    cp(fr.v_t, v_, n3);
    cp(fr.qtil, qtil_, n3);
    cp(fr.qprev, qprev_, n3);
    cp(fr.qstar, qcur_, n3);
    cp(fr.cache, cache_, 24 * ne);
  }
  if (segs_ > 1) hdk_check(hdk_seg_commit(&dseg_, ctl_, qcur_, scene_.solver.h, q_, v_, st_), "commit");
  else hdk_check(hdk_commit(static_cast<int>(n3), ctl_, qcur_, scene_.solver.h, q_, v_, st_), "commit");
  phase_mark(1);
  if (contact_scene)
    cuda_check(cudaMemcpyAsync(h_cnt_, cw_.view.cnt, sizeof(int) * HDK_CNT_INTS, cudaMemcpyDeviceToHost, st_),
               "contact counts");
  sync_ctl();
  if (contact_scene && h_ctl_->err == HDK_ERR_CAPACITY) {
    // more contacts than the working set holds: nothing was committed; grow and re-run
    ensure_contact_capacity(h_cnt_[HDK_CNT_NEED_C], h_cnt_[HDK_CNT_NEED_K], h_cnt_[HDK_CNT_NEED_U]);
    step();
    return;
  }
  phase_collect(0, 1);
  int iters = h_ctl_->iterations;
  if (segs_ > 1) {  // lockstep: the loop ran until the slowest sample finished
    seg_iterations.resize(segs_);
    seg_converged.resize(segs_);
    for (int k = 0; k < segs_; ++k) {
      seg_iterations[k] = h_ctl_[k].iterations;
      seg_converged[k] = h_ctl_[k].converged;
      iters = std::max(iters, h_ctl_[k].iterations);
      seg_sample_iterations += h_ctl_[k].iterations;
    }
  }
  if (contact_scene) {
    cw_.nc = h_cnt_[HDK_CNT_NC];
    cw_.nf = h_cnt_[HDK_CNT_NF];
    cw_.k = h_cnt_[HDK_CNT_K];
    cw_.nu = h_cnt_[HDK_CNT_NU];
    trace_iters_ = std::min(iters, ctr_.cap);
    const int spikes = (cw_.nu + 2) / 3;
    solve_count += iters + spikes;
    kernel_launches += fc_kernels_[0] + static_cast<long long>(fc_kernels_[1]) * spikes + fc_kernels_[2] +
                       static_cast<long long>(fc_kernels_[3]) * iters + fc_kernels_[4] + 1;
  } else {
    solve_count += iters;
    kernel_launches += fk_pre_ + static_cast<long long>(fk_body_) * iters + fk_post_ + 1;
  }
  check_ctl("forward step");
  last_iterations = iters;
  last_converged = h_ctl_->converged;
  for (int k = 1; k < segs_; ++k) last_converged = last_converged && h_ctl_[k].converged;
  last_contacts = contact_scene ? cw_.nc : 0;
  cur_has_contacts_ = contact_scene && cw_.k > 0;
  if (rec) {
    Frame& fr = slots_[slot];
    fr.has_contacts = cur_has_contacts_;
    if (cur_has_contacts_) {  // the adjoint's copy of this step's contact set
      if (!fr.contacts) fr.contacts = std::make_shared<ContactFrame>();
      ContactFrame& c = *fr.contacts;
      c.allocate(cw_.view.cap_c, cw_.view.cap_k, cw_.view.cap_u, cw_.view.n);
      cuda_check(cudaMemcpyAsync(c.base, cw_.base, cw_.bytes, cudaMemcpyDeviceToDevice, st_), "record contacts");
      c.nc = cw_.nc;
      c.nf = cw_.nf;
      c.k = cw_.k;
      c.nu = cw_.nu;
    }
  }
  time_ += scene_.solver.h;
  if (recording_ && force_slot_ < 0) ++nrec_;
}

void Engine::step_into(int slot) {
  if (slot < 0) raise(Code::InvalidArgument, "step_into: negative frame slot");
  force_slot_ = slot;
  try {
    step();
  } catch (...) {
    force_slot_ = -1;
    throw;
  }
  force_slot_ = -1;
}

void Engine::add_slot() {
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv), ne = scene_.mesh.ne;
  auto a = std::make_unique<DevArena>();
  Frame f;
  f.q_t = a->alloc<double>(n3);
  f.v_t = a->alloc<double>(n3);
  f.qtil = a->alloc<double>(n3);
  f.qprev = a->alloc<double>(n3);
  f.qstar = a->alloc<double>(n3);
  f.cache = a->alloc<double>(24 * ne);
  frame_mem_.push_back(std::move(a));
  slots_.push_back(f);
}

void Engine::reserve_frames(int frames) {
  while (static_cast<int>(slots_.size()) < frames) add_slot();
}

void Engine::record(bool on) {
  recording_ = on;
  if (!on) nrec_ = 0;
}

void Engine::set_state(const double* q, const double* v, double time, bool keep_frames) {
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  if (q) cuda_check(cudaMemcpyAsync(q_, q, n3 * sizeof(double), cudaMemcpyHostToDevice, st_), "set q");
  if (v) cuda_check(cudaMemcpyAsync(v_, v, n3 * sizeof(double), cudaMemcpyHostToDevice, st_), "set v");
  cuda_check(cudaStreamSynchronize(st_), "set state");
  time_ = time;
  if (!keep_frames) nrec_ = 0;
}

void Engine::set_external_force(const double* f) {
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  cuda_check(cudaMemcpyAsync(fext_, f, n3 * sizeof(double), cudaMemcpyHostToDevice, st_), "set f_ext");
  cuda_check(cudaStreamSynchronize(st_), "set f_ext");
}

void Engine::external_force_into(double* out) const {
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  cuda_check(cudaMemcpyAsync(out, fext_, n3 * sizeof(double), cudaMemcpyDeviceToHost, st_), "get f_ext");
  cuda_check(cudaStreamSynchronize(st_), "get f_ext");
}

void Engine::reset_state() { set_state(scene_.q0.data(), scene_.v0.data(), 0.0); }

Vec Engine::positions() const {
  Vec out(3 * static_cast<size_t>(scene_.mesh.nv));
  cuda_check(cudaMemcpyAsync(out.data(), q_, out.size() * sizeof(double), cudaMemcpyDeviceToHost, st_), "read state");
  cuda_check(cudaStreamSynchronize(st_), "read state");
  return out;
}
void Engine::positions_into(double* host) const {
  cuda_check(cudaMemcpyAsync(host, q_, dof_count() * sizeof(double), cudaMemcpyDeviceToHost, st_), "read state");
  cuda_check(cudaStreamSynchronize(st_), "read state");
}
void Engine::velocities_into(double* host) const {
  cuda_check(cudaMemcpyAsync(host, v_, dof_count() * sizeof(double), cudaMemcpyDeviceToHost, st_), "read state");
  cuda_check(cudaStreamSynchronize(st_), "read state");
}
Vec Engine::velocities() const {
  Vec out(3 * static_cast<size_t>(scene_.mesh.nv));
  cuda_check(cudaMemcpyAsync(out.data(), v_, out.size() * sizeof(double), cudaMemcpyDeviceToHost, st_), "read state");
  cuda_check(cudaStreamSynchronize(st_), "read state");
  return out;
}

size_t Engine::dw_count() const { return (mat_.kind == Kind::Corotated ? 2 : 1) * static_cast<size_t>(scene_.mesh.ne); }

GradOut Engine::backward(const double* direct, const double* dq_final, const double* dv_final, bool canonical,
                         bool download, const double* d_target, const GradSinks* sinks) {
  const int T = nrec_;
  if (T == 0) raise(Code::InvalidArgument, "hd_sim_backward: no recorded frames");
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv), ne = scene_.mesh.ne;
  const size_t B = n3 * sizeof(double);
  const auto h2d = [&](double* d, const double* h) {
    if (h) cuda_check(cudaMemcpyAsync(d, h, B, cudaMemcpyHostToDevice, st_), "seed upload");
    else cuda_check(cudaMemsetAsync(d, 0, B, st_), "seed zero");
  };
  if (canonical) {  // L = 1/2 |q_T - rest|^2 + 1/2 |v_T|^2, seeds from device state
    hdk_check(hdk_axpby(static_cast<int>(n3), 1.0, q_, -1.0, d_target ? d_target : rest_, qbar_, st_),
              "canonical q seed");
    hdk_check(hdk_axpby(static_cast<int>(n3), d_target ? 0.0 : 1.0, v_, 0.0, nullptr, vbar_, st_),
              "canonical v seed");
    kernel_launches += 2;
  } else {
    h2d(qbar_, direct ? direct + static_cast<size_t>(T) * n3 : dq_final);
    h2d(vbar_, dv_final);
  }
  cuda_check(cudaMemsetAsync(dfacc_, 0, B, st_), "zero");
  cuda_check(cudaMemsetAsync(dlw_, 0, 2 * ne * sizeof(double), st_), "zero");
  cuda_check(cudaMemsetAsync(dle_, 0, ne * sizeof(double), st_), "zero");
  cuda_check(cudaMemsetAsync(direct_, 0, B, st_), "zero");
  GradOut out;
  out.tau.assign(T, 1.0);
  out.rho.assign(T, 1.0);
  for (int t = T - 1; t >= 0; --t) {
    load_frame(t);
    if (direct) cuda_check(cudaMemcpyAsync(direct_, direct + static_cast<size_t>(t) * n3, B, cudaMemcpyHostToDevice, st_), "direct");
    backward_frame(t, out);
  }
  if (!download && !sinks) return out;
  const auto d2h = [&](double* h, const double* d, size_t n) {
    if (h) cuda_check(cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, st_), "grad download");
  };
  if (sinks) {
    d2h(sinks->dq0, qbar_, n3);
    d2h(sinks->dv0, vbar_, n3);
    d2h(sinks->df_ext, dfacc_, n3);
    d2h(sinks->de, dle_, ne);
    d2h(sinks->dw, dlw_, dw_count());
  } else {
    out.dl_dq0.resize(n3);
    out.dl_dv0.resize(n3);
    out.dl_df_ext.resize(n3);
    out.dl_de.resize(ne);
    out.dl_dw.resize(dw_count());
    d2h(out.dl_dq0.data(), qbar_, n3);
    d2h(out.dl_dv0.data(), vbar_, n3);
    d2h(out.dl_df_ext.data(), dfacc_, n3);
    d2h(out.dl_de.data(), dle_, ne);
    d2h(out.dl_dw.data(), dlw_, dw_count());
  }
  cuda_check(cudaStreamSynchronize(st_), "grad download");
  return out;
}

void Engine::load_frame(int t) {
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv), ne = scene_.mesh.ne;
  const Frame& f = slots_[t];
  const auto cp = [&](double* d, const double* s, size_t n) {
    cuda_check(cudaMemcpyAsync(d, s, n * sizeof(double), cudaMemcpyDeviceToDevice, st_), "frame copy");
  };
  cp(bq_t_, f.q_t, n3);
  cp(bv_t_, f.v_t, n3);
  cp(bqtil_, f.qtil, n3);
  cp(bqprev_, f.qprev, n3);
  cp(bqstar_, f.qstar, n3);
  cp(bcache_, f.cache, 24 * ne);
}

GradOut Engine::backward_slot(int slot, const double* dq_next, const double* dv_next) {
  if (slot < 0 || slot >= static_cast<int>(slots_.size()))
    raise(Code::InvalidArgument, "backward_step: the cache's frame slot is not recorded");
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv), ne = scene_.mesh.ne;
  const size_t B = n3 * sizeof(double);
  const auto h2d = [&](double* d, const double* h) {
    if (h) cuda_check(cudaMemcpyAsync(d, h, B, cudaMemcpyHostToDevice, st_), "seed upload");
    else cuda_check(cudaMemsetAsync(d, 0, B, st_), "seed zero");
  };
  h2d(qbar_, dq_next);
  h2d(vbar_, dv_next);
  cuda_check(cudaMemsetAsync(dfacc_, 0, B, st_), "zero");
  cuda_check(cudaMemsetAsync(dlw_, 0, 2 * ne * sizeof(double), st_), "zero");
  cuda_check(cudaMemsetAsync(dle_, 0, ne * sizeof(double), st_), "zero");
  cuda_check(cudaMemsetAsync(direct_, 0, B, st_), "zero");
  GradOut out;
  out.tau.assign(slots_.size(), 1.0);
  out.rho.assign(slots_.size(), 1.0);
  load_frame(slot);
  backward_frame(slot, out);
  out.tau = {out.tau[slot]};
  out.rho = {out.rho[slot]};
  out.dl_dq0.resize(n3);
  out.dl_dv0.resize(n3);
  out.dl_df_ext.resize(n3);
  out.dl_de.resize(ne);
  out.dl_dw.resize(dw_count());
  const auto d2h = [&](double* h, const double* d, size_t n) {
    cuda_check(cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, st_), "grad download");
  };
  d2h(out.dl_dq0.data(), qbar_, n3);
  d2h(out.dl_dv0.data(), vbar_, n3);
  d2h(out.dl_df_ext.data(), dfacc_, n3);
  d2h(out.dl_de.data(), dle_, ne);
  d2h(out.dl_dw.data(), dlw_, dw_count());
  cuda_check(cudaStreamSynchronize(st_), "grad download");
  return out;
}

Vec Engine::frame_vector(int slot, int which) const {
  if (slot < 0 || slot >= static_cast<int>(slots_.size())) raise(Code::InvalidArgument, "frame slot not recorded");
  Vec out(dof_count());
  const double* src = which == 0 ? slots_[slot].qtil : slots_[slot].qprev;
  cuda_check(cudaMemcpyAsync(out.data(), src, out.size() * sizeof(double), cudaMemcpyDeviceToHost, st_), "frame read");
  cuda_check(cudaStreamSynchronize(st_), "frame read");
  return out;
}

void Engine::set_eps_tr(double eps_tr) {
  if (eps_tr == eps_tr_) return;
  eps_tr_ = eps_tr;
  cuda_check(cudaStreamSynchronize(st_), "sync");
  build_backward_graph();
}

Vec Engine::solve_free(const double* rhs, const double* fixed_q) {
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  // on the engine's (non-blocking) stream: the legacy-stream cudaMemcpy would
  // not order against it
  cuda_check(cudaMemcpyAsync(seed_, rhs, n3 * sizeof(double), cudaMemcpyHostToDevice, st_), "rhs");
  if (fixed_q) cuda_check(cudaMemcpyAsync(t_, fixed_q, n3 * sizeof(double), cudaMemcpyHostToDevice, st_), "fixed q");
  else cuda_check(cudaMemsetAsync(t_, 0, n3 * sizeof(double), st_), "fixed q");
  hdk_check(hdk_gather_perm(&dv_, seed_, nullptr, rhs_, st_), "rhs gather");
  if (!hf_.fixed.empty()) {
    hdk_check(hdk_fixed_coupling(&a_fd_, d_fixed_, t_, fixc_, st_), "coupling");
    hdk_check(hdk_axpby(3 * hf_.n, 1.0, rhs_, -1.0, fixc_, rhs_, st_), "rhs - A_fd q_d");
  }
  hdk_check(hdk_apply_inverse3(&df_, rhs_, t_, st_), "solve");
  ++solve_count;
  Vec out(n3);
  cuda_check(cudaMemcpyAsync(out.data(), t_, n3 * sizeof(double), cudaMemcpyDeviceToHost, st_), "download");
  cuda_check(cudaStreamSynchronize(st_), "sync");
  return out;
}

double Engine::time_solve(int reps, double* bytes) {
  cudaEvent_t a, b;
  cuda_check(cudaEventCreate(&a), "event");
  cuda_check(cudaEventCreate(&b), "event");
  for (int i = 0; i < 2; ++i) hdk_check(hdk_apply_inverse3_perm(&df_, rhs_, dqp_, st_), "warm solve");
  cuda_check(cudaEventRecord(a, st_), "event");
  for (int i = 0; i < reps; ++i) hdk_check(hdk_apply_inverse3_perm(&df_, rhs_, dqp_, st_), "timed solve");
  cuda_check(cudaEventRecord(b, st_), "event");
  cuda_check(cudaEventSynchronize(b), "event sync");
  float ms = 0;
  cuda_check(cudaEventElapsedTime(&ms, a, b), "elapsed");
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  kernel_launches += 4LL * (reps + 2);
  // factor values streamed by both passes + rhs read, z write/read, x write
  if (bytes) *bytes = 16.0 * static_cast<double>(hf_.row_off.back()) + 96.0 * hf_.n;
  return static_cast<double>(ms) / reps;
}

namespace {
// Same factor structure (ordering, pattern, stream layout, A_ff / A_fd
// patterns): only values differ, so the device buffers can be refilled.
bool same_structure(const HostFactor& a, const HostFactor& b) {
  const auto eq_bytes = [](const auto& x, const auto& y) {
    return x.size() == y.size() && (x.empty() || std::memcmp(x.data(), y.data(), sizeof(x[0]) * x.size()) == 0);
  };
  return a.n == b.n && a.stream_len == b.stream_len && a.p2v == b.p2v && a.row_pslot == b.row_pslot &&
         eq_bytes(a.sdesc, b.sdesc) && eq_bytes(a.chunks, b.chunks) && a.tile_chunk == b.tile_chunk &&
         a.a_ff.off == b.a_ff.off && a.a_ff.col == b.a_ff.col && a.a_fd.off == b.a_fd.off && a.a_fd.col == b.a_fd.col;
}
}  // namespace

void Engine::set_young(const Vec& young, bool freeze) {
  const auto t0 = std::chrono::steady_clock::now();
  if (freeze) mat_.freeze();
  if (segs_ > 1) segmented_set_young(mat_, young, scene_.mesh.vol, segs_);
  else mat_.set_young(young, scene_.mesh.vol);
  cuda_check(cudaStreamSynchronize(st_), "sync");
  if (refactor_on_device()) {
    // same pattern, ordering and stream layout: values only, all on the device
    const auto lap = [&t0] {
      return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    const double t_mat = lap();
    upload_material();
    const double t_up = lap();
    refactor_device_values();
    const double t_num = lap();
    ++refactor_count;
    cols_.reset();
    nrec_ = 0;  // recorded frames are stale; their slots (sized by the mesh) are reused
    build_forward_graph();
    build_backward_graph();
    last_refactor_device = true;
    last_refactor_ms = lap();
    if (const char* tr = std::getenv("HETERODYN_REFACTOR_TRACE"); tr && std::atoi(tr) != 0)
      std::fprintf(stderr, "[refactor] material %.2f ms, upload %.2f ms, device numeric %.2f ms, graphs %.2f ms\n",
                   t_mat, t_up - t_mat, t_num - t_up, last_refactor_ms - t_num);
    return;
  }
  last_refactor_device = false;
  HostFactor nf = build_factor(scene_.mesh, mat_, scene_.solver.h, scene_.fixed, scene_.ordering, device_values_,
                               &order_cache_, &hf_);
  ++refactor_count;
  cols_.reset();  // its graph bakes the old factor and material pointers
  if (same_structure(hf_, nf)) {
    // values only: refill the existing buffers, keep every allocation, and
    // re-capture the graphs (they bake the material scalars by value)
    hf_ = std::move(nf);
    upload_material();
    fill_factor_values(const_cast<double*>(df_.sval));
    refresh_fp32();
    DevArena::copy_h2d(const_cast<double*>(a_ff_.val), hf_.a_ff.val.data(), hf_.a_ff.val.size() * sizeof(double));
    if (!hf_.a_fd.val.empty()) {
      DevArena::copy_h2d(const_cast<double*>(a_fd_.val), hf_.a_fd.val.data(), hf_.a_fd.val.size() * sizeof(double));
      Vec tv(hf_.a_fd.val.size());  // A_df = A_fd^T values, in the transpose's order
      std::vector<int> cur(hf_.a_fd.cols + 1, 0);
      for (int c : hf_.a_fd.col) ++cur[c + 1];
      for (int r = 0; r < hf_.a_fd.cols; ++r) cur[r + 1] += cur[r];
      for (int p = 0; p < hf_.a_fd.rows; ++p)
        for (int k = hf_.a_fd.off[p]; k < hf_.a_fd.off[p + 1]; ++k) tv[cur[hf_.a_fd.col[k]]++] = hf_.a_fd.val[k];
      DevArena::copy_h2d(const_cast<double*>(a_df_.val), tv.data(), tv.size() * sizeof(double));
    }
    nrec_ = 0;  // recorded frames are stale; their slots (sized by the mesh) are reused
    build_forward_graph();
    build_backward_graph();
    return;
  }
  hf_ = std::move(nf);
  // material arrays and factor live in fresh allocations; graphs bake pointers
  // (the state and any f_ext set through hd_sim_set_external_force survive)
  Vec q = positions(), v = velocities(), f(dof_count());
  external_force_into(f.data());
  const double t = time_;
  build_static();
  build_factor_device();
  set_state(q.data(), v.data(), t);
  set_external_force(f.data());
  nrec_ = 0;  // recorded frames are stale; their slots (sized by the mesh) are reused
  build_forward_graph();
  build_backward_graph();
}

}  // namespace hdb
