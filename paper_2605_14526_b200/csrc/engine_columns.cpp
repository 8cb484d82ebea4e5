// Contact adjoint columns, several at a time (reference backward.cpp:229-238:
// x_c = (A - B)^{-1} j_c warm-started from the cached A^{-1} j_c, one
// backbone fixed point per contact row).  Each column runs exactly the
// single-column backbone of engine.cpp (same kernels, same Anderson state
// layout, its own control block), but the global solve of all kColumns
// columns is one multi-column stream of the factor (hdk_apply_inverse3_multi),
// and the columns' vector kernels run on their own streams between two
// solves.  The loop runs while any column is active; a column past
// convergence skips its kernels (its control block's cond is 0).
#include "engine.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace hdb {

static void hdk_ok(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

struct Engine::ColumnSet {
  struct Col {
    hdk_ctl* ctl = nullptr;  // = ctls + c
    hdk_ctl* snap = nullptr;
    void* res = nullptr;
    double *seed = nullptr, *x = nullptr, *seedp = nullptr, *xp = nullptr, *t = nullptr, *tv = nullptr;
    double *lastq = nullptr, *lastg = nullptr, *dq = nullptr, *dg = nullptr;
    double *rt = nullptr, *rx = nullptr, *lrx = nullptr, *lrg = nullptr, *rsq = nullptr, *ef = nullptr, *part = nullptr;
    hdk_factor f{};  // the multi-column factor view of this column (part2 offset)
    cudaStream_t s1 = nullptr, s2 = nullptr;
    cudaEvent_t fork = nullptr, mid = nullptr, join = nullptr, end = nullptr;
  };
  std::unique_ptr<DevArena> mem;
  hdk_factor f{};  // df_ with kColumns columns of solve scratch
  Col col[kColumns];
  hdk_ctl* ctls = nullptr;
  hdk_ctl* h_ctls = nullptr;  // pinned mirror
  double* rhs = nullptr;      // kColumns x 3n
  int* any = nullptr;         // OR of the columns' cond
  int* h_any = nullptr;
  LoopGraph graph;
  LoopGraph rgraph;          // refill loop: one iteration per body, exits when a column finishes
  int* expected = nullptr;   // columns iterating at launch (device)
  int* h_expected = nullptr;
  hdk_bb_columns bb{};  // every column's backbone buffers, for the one-launch-per-stage body
  // Column-batched CG (the default backbone, engine_pcg.cpp's algorithm per
  // column): the columns' seed / x by vertex, their seedp / xp / R(x0) in
  // elimination order and their element forces are contiguous [kColumns][..]
  // (Col's pointers index into them); r is rhs.
  double *seed_all = nullptr, *x_all = nullptr, *seedp_all = nullptr, *xp_all = nullptr, *rx_all = nullptr,
         *ef_all = nullptr;
  double *cz = nullptr, *cp = nullptr, *cq = nullptr, *cax = nullptr, *cpv = nullptr, *cpart = nullptr;
  hdk_pcg* cst = nullptr;
  hdk_pcg* h_cst = nullptr;
  unsigned int* ctickets = nullptr;
  LoopGraph pgraph;
  // block CG (default): the batch's columns in one block Krylov space
  hdk_bcg* bst = nullptr;
  double* dpart = nullptr;  // column deflation partials / tickets
  unsigned int* dtickets = nullptr;
  hdk_bcg* h_bst = nullptr;
  int* bm = nullptr;
  int* h_bm = nullptr;
  double* bpart = nullptr;
  unsigned int* bticket = nullptr;
  LoopGraph bgraph;
  double* cg_trace = nullptr;  // profiling (HETERODYN_CG_TRACE)
  double** h_cg_trace_ptr = nullptr;
  const char* cg_trace_path = nullptr;
  long long* trace = nullptr;  // profiling (HETERODYN_CHUNK_TRACE)
  long long** h_trace_ptr = nullptr;
  const char* trace_path = nullptr;
  int trace_grid = 0, trace_chunks = 0;
  std::vector<int> h_first2;
  ~ColumnSet() {
    if (cg_trace) {
      std::vector<double> h(static_cast<size_t>(kColumns) * 512 * 2);
      if (cudaMemcpy(h.data(), cg_trace, h.size() * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess)
        if (FILE* fp = std::fopen(cg_trace_path, "wb")) {
          std::fwrite(h.data(), sizeof(double), h.size(), fp);
          std::fclose(fp);
        }
      cudaFree(cg_trace);
      cudaFreeHost(h_cg_trace_ptr);
    }
    if (trace) {
      std::vector<long long> h(4 * static_cast<size_t>(trace_chunks));
      if (cudaMemcpy(h.data(), trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess) {
        if (FILE* fp = std::fopen(trace_path, "wb")) {
          std::fwrite(&trace_grid, sizeof(int), 1, fp);
          std::fwrite(h_first2.data(), sizeof(int), h_first2.size(), fp);
          std::fwrite(h.data(), sizeof(long long), h.size(), fp);
          std::fclose(fp);
        }
      }
      cudaFree(trace);
      cudaFreeHost(h_trace_ptr);
    }
    pgraph.destroy();
    pgraph.destroy();
    bgraph.destroy();
    if (h_bst) cudaFreeHost(h_bst);
    if (h_bm) cudaFreeHost(h_bm);
    if (h_cst) cudaFreeHost(h_cst);
    graph.destroy();
    rgraph.destroy();
    if (h_expected) cudaFreeHost(h_expected);
    for (Col& c : col) {
      for (cudaEvent_t e : {c.fork, c.mid, c.join, c.end})
        if (e) cudaEventDestroy(e);
      for (cudaStream_t st : {c.s1, c.s2})
        if (st) cudaStreamDestroy(st);
    }
    if (h_ctls) cudaFreeHost(h_ctls);
    if (h_any) cudaFreeHost(h_any);
  }
};

void Engine::ColumnSetDeleter::operator()(ColumnSet* p) const { delete p; }

void Engine::build_columns() {
  cols_.reset(new ColumnSet());
  ColumnSet& S = *cols_;
  S.mem = std::make_unique<DevArena>();
  DevArena& A = *S.mem;
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv), n3p = 3 * static_cast<size_t>(hf_.n),
               ne = scene_.mesh.ne;
  S.f = df_;
  S.f.part1 = A.alloc<double>(kColumns * 3 * static_cast<size_t>(df_.n_pslot));
  S.f.z = A.alloc<double>(kColumns * n3p);
  const size_t p2 = hdk_factor_part2_stride(&df_);
  S.f.part2 = A.alloc<double>(kColumns * p2);
  S.ctls = A.alloc<hdk_ctl>(kColumns);
  S.rhs = A.alloc<double>(kColumns * n3p);
  S.any = A.alloc<int>(1);
  S.expected = A.alloc<int>(1);
  cuda_check(cudaMallocHost(&S.h_expected, sizeof(int)), "pinned expected");
  S.f.run_flag = S.any;
  cuda_check(cudaMallocHost(&S.h_ctls, sizeof(hdk_ctl) * kColumns), "pinned ctl");
  cuda_check(cudaMallocHost(&S.h_any, sizeof(int)), "pinned flag");
  S.seed_all = A.alloc<double>(kColumns * n3);
  S.x_all = A.alloc<double>(kColumns * n3);
  S.seedp_all = A.alloc<double>(kColumns * n3p);
  S.xp_all = A.alloc<double>(kColumns * n3p);
  S.rx_all = A.alloc<double>(kColumns * n3p);
  S.ef_all = A.alloc<double>(kColumns * 12 * ne);
  for (int c = 0; c < kColumns; ++c) {
    ColumnSet::Col& C = S.col[c];
    C.ctl = S.ctls + c;
    C.snap = A.alloc<hdk_ctl>(1);
    C.res = A.raw(hdk_bb_result_bytes());
    C.seed = S.seed_all + c * n3;
    C.x = S.x_all + c * n3;
    C.tv = A.alloc<double>(n3);
    C.seedp = S.seedp_all + c * n3p;
    C.xp = S.xp_all + c * n3p;
    C.rx = S.rx_all + c * n3p;
    for (double** v : {&C.t, &C.lastq, &C.lastg, &C.rt, &C.lrx, &C.lrg}) *v = A.alloc<double>(n3p);
    C.dq = A.alloc<double>(HDK_AA_MAX * n3p);
    C.dg = A.alloc<double>(HDK_AA_MAX * n3p);
    C.rsq = A.alloc<double>(HDK_AA_MAX * n3p);
    C.ef = S.ef_all + c * 12 * ne;
    C.part = A.alloc<double>(HDK_RED_BLOCKS * HDK_RED_Q);
    C.f = S.f;
    C.f.part2 = S.f.part2 + c * p2;
    C.f.run_flag = nullptr;
    cuda_check(cudaStreamCreateWithFlags(&C.s1, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&C.s2, cudaStreamNonBlocking), "stream");
    for (cudaEvent_t* e : {&C.fork, &C.mid, &C.join, &C.end})
      cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
  }
  static_assert(kColumns == HDK_BB_COLUMNS, "column batch width");
  for (int c = 0; c < kColumns; ++c) {
    const ColumnSet::Col& C = S.col[c];
    hdk_bb_column& k = S.bb.col[c];
    k.f = C.f;
    k.ctl = C.ctl;
    k.snap = C.snap;
    k.res = C.res;
    k.t = C.t;
    k.tv = C.tv;
    k.xp = C.xp;
    k.x = C.x;
    k.lastq = C.lastq;
    k.lastg = C.lastg;
    k.dq = C.dq;
    k.dg = C.dg;
    k.part = C.part;
    k.rt = C.rt;
    k.rx = C.rx;
    k.lrx = C.lrx;
    k.lrg = C.lrg;
    k.rsq = C.rsq;
    k.ef = C.ef;
    k.rhs = S.rhs + c * 3 * static_cast<size_t>(hf_.n);
    k.seedp = C.seedp;
  }
  void* s = st_;
  // first right-hand sides seed + R(x0) of every column
  auto pre = [&] {
    for (int c = 0; c < kColumns; ++c) {
      ColumnSet::Col& C = S.col[c];
      hdk_ok(hdk_aa_reset(C.ctl, HDK_AA_MAX, 1e8, 500, 1e-10, s), "aa reset");
      hdk_ok(hdk_gather_perm(&dv_, C.seed, nullptr, C.seedp, s), "seed in elimination order");
      hdk_ok(hdk_gather_perm(&dv_, C.x, nullptr, C.xp, s), "x0 in elimination order");
      hdk_ok(hdk_bapply(&dm_, dcomp_, C.x, C.ef, s), "B x0");
      hdk_ok(hdk_gather_pp(&dv_, nullptr, C.ef, C.rx, nullptr, s), "R(x0)");
      hdk_ok(hdk_axpby(static_cast<int>(n3p), 1.0, C.seedp, 1.0, C.rx, S.rhs + c * n3p, s), "rhs0");
    }
    hdk_ok(hdk_any_cond(S.ctls, kColumns, S.any, 0ULL, s), "any");
  };
  auto body = [&](unsigned long long handle) {
    for (int u = 0; u < unroll_; ++u) columns_body(handle, 0u);
  };
  build_loop_graph(st_, use_cond_, pre, body, [] {}, S.graph);
  // refill loop: no pre (slots are initialised one by one), one iteration per body
  auto rbody = [&](unsigned long long handle) { columns_body(handle, 4u); };
  build_loop_graph(st_, use_cond_, [] {}, rbody, [] {}, S.rgraph);
}

// First right-hand side seed + R(x0) of one slot (the pre step of the loop, per column).
void Engine::column_pre(int j) {
  ColumnSet& S = *cols_;
  ColumnSet::Col& C = S.col[j];
  void* s = st_;
  const size_t n3p = 3 * static_cast<size_t>(hf_.n);
  hdk_ok(hdk_aa_reset(C.ctl, HDK_AA_MAX, 1e8, 500, 1e-10, s), "aa reset");
  hdk_ok(hdk_gather_perm(&dv_, C.seed, nullptr, C.seedp, s), "seed in elimination order");
  hdk_ok(hdk_gather_perm(&dv_, C.x, nullptr, C.xp, s), "x0 in elimination order");
  hdk_ok(hdk_bapply(&dm_, dcomp_, C.x, C.ef, s), "B x0");
  hdk_ok(hdk_gather_pp(&dv_, nullptr, C.ef, C.rx, nullptr, s), "R(x0)");
  hdk_ok(hdk_axpby(static_cast<int>(n3p), 1.0, C.seedp, 1.0, C.rx, S.rhs + j * n3p, s), "rhs0");
  kernel_launches += 6;
}

int Engine::solve_all_columns(const ContactFrame& c) {
  if (!cols_) build_columns();
  ColumnSet& S = *cols_;
  const int nv = scene_.mesh.nv;
  const size_t n3 = 3 * static_cast<size_t>(nv);
  int slot_row[kColumns];
  int next = 0, active = 0, iters = 0;
  const auto assign = [&](int j) {
    if (next < c.k) {
      slot_row[j] = next;
      hdk_ok(hdk_contact_column_init(&c.view, next, nv, df_.v2p, S.col[j].seed, S.col[j].x, st_), "column init");
      column_pre(j);
      ++next;
      ++active;
    } else {
      slot_row[j] = -1;
      cuda_check(cudaMemsetAsync(&S.col[j].ctl->cond, 0, sizeof(int), st_), "idle slot");
    }
  };
  for (int j = 0; j < kColumns; ++j) assign(j);
  if (ph_.on) cuda_check(cudaEventRecord(ph_.ev[6], st_), "phase event");
  long long rounds = 0;
  while (active > 0) {
    *S.h_expected = active;
    cuda_check(cudaMemcpyAsync(S.expected, S.h_expected, sizeof(int), cudaMemcpyHostToDevice, st_), "expected");
    const int one = 1;
    cuda_check(cudaMemcpyAsync(S.any, &one, sizeof(int), cudaMemcpyHostToDevice, st_), "run flag");
    if (S.rgraph.exec) {
      cuda_check(cudaGraphLaunch(S.rgraph.exec, st_), "columns");
    } else {  // host-driven loop (profiling fallback)
      for (;;) {
        cuda_check(cudaGraphLaunch(S.rgraph.body, st_), "columns");
        cuda_check(cudaMemcpyAsync(S.h_any, S.any, sizeof(int), cudaMemcpyDeviceToHost, st_), "flag");
        cuda_check(cudaStreamSynchronize(st_), "sync");
        if (!*S.h_any) break;
      }
    }
    ++rounds;
    cuda_check(cudaMemcpyAsync(S.h_ctls, S.ctls, sizeof(hdk_ctl) * kColumns, cudaMemcpyDeviceToHost, st_), "ctl read");
    cuda_check(cudaStreamSynchronize(st_), "columns sync");
    for (int j = 0; j < kColumns; ++j) {
      if (slot_row[j] < 0) continue;
      hdk_ctl& h = S.h_ctls[j];
      if (h.err == 0 && h.nonfinite) h.err = 10;
      if (h.err != 0) {
        std::memcpy(h_ctl_, &h, sizeof(hdk_ctl));
        check_ctl("backward step (contact column)");
      }
      if (h.cond != 0) continue;  // still iterating
      iters += h.iterations;
      ph_.col_real_iters += h.iterations;
      cuda_check(cudaMemcpyAsync(cX_ + n3 * slot_row[j], S.col[j].x, n3 * sizeof(double), cudaMemcpyDeviceToDevice,
                                 st_), "column");
      --active;
      assign(j);
    }
  }
  if (ph_.on) {
    cuda_check(cudaEventRecord(ph_.ev[7], st_), "phase event");
    cuda_check(cudaEventSynchronize(ph_.ev[7]), "phase event");
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ph_.ev[6], ph_.ev[7]) == cudaSuccess) ph_.col_ms += ms;
  }
  kernel_launches += static_cast<long long>(S.rgraph.counts[1]) * (iters / kColumns + rounds);
  ph_.col_batches += rounds;
  column_solves += iters;
  column_streams += iters / kColumns + rounds;
  return iters;
}

// One multi-column iteration; skip bits (profiling): 1 solve, 2 column kernels;
// bit 4: the refill loop's condition (exit when a column finishes).
void Engine::columns_body(unsigned long long handle, unsigned skip) {
  ColumnSet& S = *cols_;
  void* s = st_;
  const size_t n3p = 3 * static_cast<size_t>(hf_.n);
  {
    {
      if (!(skip & 1u)) hdk_ok(hdk_apply_inverse3_multi(&S.f, S.rhs, kColumns, s), "multi-column solve");
      static const bool batched = [] {
        const char* e = std::getenv("HETERODYN_COLVEC");  // "0": one stream pair per column (A/B)
        return !(e && e[0] == '0');
      }();
      if (batched && !(skip & 2u)) {
        // one launch per backbone stage for all columns; the coefficient
        // solves run on a second branch beside B t and its gather
        ColumnSet::Col& C0 = S.col[0];
        hdk_ok(hdk_bb_columns_dots(&S.bb, 1, s), "dots (columns)");
        cuda_check(cudaEventRecord(C0.mid, st_), "mid");
        cuda_check(cudaStreamWaitEvent(C0.s2, C0.mid, 0), "mid wait");
        hdk_ok(hdk_bb_columns_solve(&S.bb, C0.s2), "coefficients (columns)");
        cuda_check(cudaEventRecord(C0.join, C0.s2), "join");
        hdk_ok(hdk_bb_columns_bapply(&dm_, dcomp_, &S.bb, s), "B t (columns)");
        hdk_ok(hdk_bb_columns_gather(&dv_, &S.bb, s), "R(t) (columns)");
        cuda_check(cudaStreamWaitEvent(st_, C0.join, 0), "join wait");
        hdk_ok(hdk_bb_columns_mix(&S.bb, s), "mix (columns)");
      }
      for (int c = 0; c < kColumns && !(skip & 2u) && !batched; ++c) {
        ColumnSet::Col& C = S.col[c];
        cuda_check(cudaEventRecord(C.fork, st_), "fork");
        cuda_check(cudaStreamWaitEvent(C.s1, C.fork, 0), "fork wait");
        hdk_ok(hdk_bb_dots(&C.f, C.ctl, C.snap, C.t, C.tv, C.xp, C.lastq, C.lastg, C.dq, C.dg, C.part, 1, C.s1), "dots");
        cuda_check(cudaEventRecord(C.mid, C.s1), "mid");
        cuda_check(cudaStreamWaitEvent(C.s2, C.mid, 0), "mid wait");
        hdk_ok(hdk_bb_solve(C.ctl, C.snap, C.part, C.res, 0ULL, C.s2), "coefficients");
        cuda_check(cudaEventRecord(C.join, C.s2), "join");
        hdk_ok(hdk_bapply_flag(&dm_, dcomp_, C.tv, C.ef, &C.snap->cond, C.s1), "B t");
        hdk_ok(hdk_gather_pp(&dv_, nullptr, C.ef, C.rt, &C.snap->cond, C.s1), "R(t)");
        cuda_check(cudaStreamWaitEvent(C.s1, C.join, 0), "join wait");
        hdk_ok(hdk_bb_mix(&C.f, C.ctl, C.snap, C.res, C.t, C.xp, C.x, C.dq, C.rt, C.rx, C.lrx, C.lrg, C.rsq, C.seedp,
                          S.rhs + c * n3p, C.s1),
               "mix");
        cuda_check(cudaEventRecord(C.end, C.s1), "end");
        cuda_check(cudaStreamWaitEvent(st_, C.end, 0), "end wait");
      }
      if (skip & 4u) hdk_ok(hdk_cols_cond(S.ctls, kColumns, S.expected, S.any, handle, s), "refill cond");
      else hdk_ok(hdk_any_cond(S.ctls, kColumns, S.any, handle, s), "any");
    }
  }
}

double Engine::time_columns(int reps, unsigned skip) {
  if (!cols_) build_columns();
  cudaGraphExec_t g = nullptr;
  {
    cudaGraph_t gr = nullptr;
    cuda_check(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal), "capture");
    columns_body(0ULL, skip);
    cuda_check(cudaStreamEndCapture(st_, &gr), "capture");
    cuda_check(cudaGraphInstantiate(&g, gr, 0), "instantiate");
    cudaGraphDestroy(gr);
  }
  cudaEvent_t a, b;
  cuda_check(cudaEventCreate(&a), "event");
  cuda_check(cudaEventCreate(&b), "event");
  for (int i = 0; i < 3; ++i) cuda_check(cudaGraphLaunch(g, st_), "warm");
  cuda_check(cudaEventRecord(a, st_), "event");
  for (int i = 0; i < reps; ++i) cuda_check(cudaGraphLaunch(g, st_), "timed");
  cuda_check(cudaEventRecord(b, st_), "event");
  cuda_check(cudaEventSynchronize(b), "sync");
  float ms = 0.f;
  cuda_check(cudaEventElapsedTime(&ms, a, b), "elapsed");
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaGraphExecDestroy(g);
  return static_cast<double>(ms) / reps;
}

// The columns' CG loop (engine_pcg.cpp's algorithm, one CG per column, every
// stage one launch for all kColumns columns): B p by column (blockIdx.y),
// q = A p - gather(B p) with p.q, x / r, the multi-column solve z = A^{-1} r
// folded per column with r.z and the stopping test, p = z + beta p.  The
// multi-column solve runs while any column iterates.
void Engine::build_columns_pcg() {
  ColumnSet& S = *cols_;
  DevArena& A = *S.mem;
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv), n3p = 3 * static_cast<size_t>(hf_.n),
               ne = scene_.mesh.ne;
  const int n = hf_.n, nv = scene_.mesh.nv, K = kColumns;
  for (double** v : {&S.cz, &S.cp, &S.cq, &S.cax}) *v = A.alloc<double>(K * n3p);
  S.cpv = A.alloc<double>(K * n3);
  cuda_zero(S.cpv, K * n3 * sizeof(double), "zero pv");  // fixed vertices stay 0
  const size_t pst = hdk_cpcg_partial_stride(n);
  S.cpart = A.alloc<double>(pst * K);
  S.cst = A.alloc<hdk_pcg>(K);
  S.ctickets = A.alloc<unsigned int>(K);
  cuda_zero(S.ctickets, sizeof(unsigned int) * K, "zero tickets");
  cuda_check(cudaMallocHost(&S.h_cst, sizeof(hdk_pcg) * K), "pinned pcg");
  void* s = st_;
  const int cstride = static_cast<int>(sizeof(hdk_pcg) / sizeof(int));
  auto pre = [&] {
    hdk_ok(hdk_spcg_init(S.cst, K, 1e-10, 500, S.any, s), "pcg init");
    for (int c = 0; c < K; ++c) {
      ColumnSet::Col& C = S.col[c];
      hdk_ok(hdk_gather_perm(&dv_, C.seed, nullptr, C.seedp, s), "seed in elimination order");
      hdk_ok(hdk_gather_perm(&dv_, C.x, nullptr, C.xp, s), "x0 in elimination order");
      hdk_ok(hdk_bapply(&dm_, dcomp_, C.x, C.ef, s), "B x0");
      hdk_ok(hdk_gather_pp(&dv_, nullptr, C.ef, C.rx, nullptr, s), "R(x0)");
    }
    hdk_ok(hdk_cpcg_spmv(&a_ff_, K, S.xp_all, S.cax, S.cst, s), "A x0");
    hdk_ok(hdk_pcg_r0(static_cast<int>(K * n3p), S.seedp_all, S.cax, S.rx_all, S.rhs, s), "r0");
    hdk_ok(hdk_apply_inverse3_multi(&S.f, S.rhs, K, s), "z0 = A^-1 r0");
    hdk_ok(hdk_cpcg_rz(&S.f, K, S.rhs, S.cz, S.xp_all, S.cpart, pst, S.ctickets, S.cst, s), "rz");
    hdk_ok(hdk_cpcg_p(n, nv, K, S.cz, S.cp, S.cpv, df_.p2v, S.cst, S.any, 0ULL, s), "p");
  };
  auto body = [&](unsigned long long handle) {
    hdk_ok(hdk_bapply_cols_sorted(&dm_, dcomp_, S.cpv, n3, S.ef_all, 12 * ne, corner_pos_, &S.cst->cond, cstride, K,
                                  s),
           "B p (columns)");
    hdk_ok(hdk_cpcg_apply(&dv_, &a_ff_, K, S.ef_all, 12 * ne, S.cp, S.cq, S.cpart, pst, S.ctickets, S.cst, s),
           "q = (A - B) p (columns)");
    hdk_ok(hdk_spcg_xr(static_cast<int>(n3p), static_cast<int>(K * n3p), S.xp_all, S.rhs, S.cp, S.cq, S.cst, s),
           "x, r (columns)");
    hdk_ok(hdk_apply_inverse3_multi(&S.f, S.rhs, K, s), "z = A^-1 r (columns)");
    hdk_ok(hdk_cpcg_rz(&S.f, K, S.rhs, S.cz, S.xp_all, S.cpart, pst, S.ctickets, S.cst, s), "rz (columns)");
    hdk_ok(hdk_cpcg_p(n, nv, K, S.cz, S.cp, S.cpv, df_.p2v, S.cst, S.any, handle, s), "p + any (columns)");
  };
  build_loop_graph(st_, use_cond_, pre, body, [] {}, S.pgraph);
}

// The batch's columns by block CG (pcg.cu hdk_bcg_*): B p and q = (A - B) p
// per column as in the column CG, then the block's Gram matrices, X / R,
// the multi-column solve, Z^T R with the per-column stopping tests, P.
void Engine::build_columns_bcg() {
  ColumnSet& S = *cols_;
  if (!S.cst) build_columns_pcg();
  DevArena& A = *S.mem;
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv), n3p = 3 * static_cast<size_t>(hf_.n),
               ne = scene_.mesh.ne;
  const int n = hf_.n, nv = scene_.mesh.nv, K = kColumns;
  S.bst = A.alloc<hdk_bcg>(1);
  S.bm = A.alloc<int>(1);
  S.bpart = A.alloc<double>(hdk_bcg_partial_doubles(n));
  S.bticket = A.alloc<unsigned int>(1);
  cuda_check(cudaMallocHost(&S.h_bst, sizeof(hdk_bcg)), "pinned bcg");
  cuda_check(cudaMallocHost(&S.h_bm, sizeof(int)), "pinned bcg");
  // deflation by the frame's recycled W (column_deflation_setup): its own partials and tickets
  if (defl_.on) defl_alloc();
  Deflation& D = defl_;
  S.dpart = A.alloc<double>(hdk_bdefl_partial_doubles(n));
  S.dtickets = A.alloc<unsigned int>(8);
  void* s = st_;
  auto pre = [&] {
    hdk_ok(hdk_bcg_init(S.bst, S.bm, 1e-10, 500, S.any, S.cst, K, s), "block CG init");
    for (int c = 0; c < K; ++c) {
      ColumnSet::Col& C = S.col[c];
      hdk_ok(hdk_gather_perm(&dv_, C.seed, nullptr, C.seedp, s), "seed in elimination order");
      hdk_ok(hdk_gather_perm(&dv_, C.x, nullptr, C.xp, s), "x0 in elimination order");
      hdk_ok(hdk_bapply(&dm_, dcomp_, C.x, C.ef, s), "B x0");
      hdk_ok(hdk_gather_pp(&dv_, nullptr, C.ef, C.rx, nullptr, s), "R(x0)");
    }
    hdk_ok(hdk_cpcg_spmv(&a_ff_, K, S.xp_all, S.cax, S.cst, s), "A x0");
    hdk_ok(hdk_pcg_r0(static_cast<int>(K * n3p), S.seedp_all, S.cax, S.rx_all, S.rhs, s), "r0");
    if (D.d) {  // Galerkin first iterates on span W
      hdk_ok(hdk_bdefl_dots(static_cast<int>(n3p), S.rhs, D.w, D.d, S.bst, S.dpart, S.dtickets, s), "W^T R0");
      hdk_ok(hdk_bdefl_correct(static_cast<int>(n3p), S.xp_all, S.rhs, D.w, D.aw, D.d, S.bst, s), "X0, R0 on span W");
    }
    hdk_ok(hdk_apply_inverse3_multi(&S.f, S.rhs, K, s), "Z0 = A^-1 R0");
    hdk_ok(hdk_bcg_zfold(&S.f, S.rhs, S.cz, S.xp_all, S.bpart, S.bticket, S.bst, s), "Z^T R");
    if (D.d) hdk_ok(hdk_bdefl_dots(static_cast<int>(n3p), S.cz, D.aw, D.d, S.bst, S.dpart, S.dtickets, s), "(AW)^T Z");
    hdk_ok(hdk_bcg_p(n, nv, S.cz, S.cp, S.cpv, df_.p2v, S.bst, S.any, D.d, D.w, 0ULL, s), "P");
  };
  const int cstride = static_cast<int>(sizeof(hdk_pcg) / sizeof(int));
  auto body = [&](unsigned long long handle) {
    hdk_ok(hdk_bapply_cols_sorted(&dm_, dcomp_, S.cpv, n3, S.ef_all, 12 * ne, corner_pos_, &S.cst->cond, cstride, K,
                                  s),
           "B P (block)");
    hdk_ok(hdk_cpcg_apply_q(&dv_, &a_ff_, K, S.ef_all, 12 * ne, S.cp, S.cq, S.cst, s), "Q = (A - B) P");
    hdk_ok(hdk_bcg_gram_pq(static_cast<int>(n3p), S.cp, S.cq, S.bpart, S.bticket, S.bst, s), "P^T Q, alpha");
    hdk_ok(hdk_bcg_xr(static_cast<int>(n3p), S.xp_all, S.rhs, S.cp, S.cq, S.bst, s), "X, R");
    hdk_ok(hdk_apply_inverse3_multi(&S.f, S.rhs, K, s), "Z = A^-1 R (block)");
    hdk_ok(hdk_bcg_zfold(&S.f, S.rhs, S.cz, S.xp_all, S.bpart, S.bticket, S.bst, s), "Z^T R, beta");
    if (D.d) hdk_ok(hdk_bdefl_dots(static_cast<int>(n3p), S.cz, D.aw, D.d, S.bst, S.dpart, S.dtickets, s), "(AW)^T Z");
    hdk_ok(hdk_bcg_p(n, nv, S.cz, S.cp, S.cpv, df_.p2v, S.bst, S.any, D.d, D.w, handle, s), "P + cond");
  };
  build_loop_graph(st_, use_cond_, pre, body, [] {}, S.bgraph);
}

// Once per contact frame, before its column batches: (A - B) W and E for this
// frame's operator from the recycled W (the backbone's deflation vectors),
// so the batches' block CG deflates too (hdk_bdefl_*); without a valid W the
// columns run plain block CG (cols = 0).
void Engine::column_deflation_setup() {
  Deflation& D = defl_;
  if (!D.d) return;
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv), n3p = 3 * static_cast<size_t>(hf_.n),
               ne = scene_.mesh.ne;
  // opt-in (HETERODYN_COLUMN_DEFLATION=1): the batch's block Krylov space
  // already holds the slow modes W would remove — C4 3,865 vs 4,019 batched
  // iterations per 8 steps, but 340 vs 317 us each
  static const bool enabled = [] {
    const char* e = std::getenv("HETERODYN_COLUMN_DEFLATION");
    return e && e[0] == '1';
  }();
  const bool on = D.on && D.valid && enabled;
  D.h->use = on ? 1 : 0;
  D.h->k = on ? D.k : 0;
  D.h->rec = 0;
  D.h->hcap = D.hcap;
  D.h->active = 0;
  D.h->cols = on ? 1 : 0;
  cuda_check(cudaMemcpyAsync(&D.d->k, &D.h->k, 6 * sizeof(int), cudaMemcpyHostToDevice, st_), "column deflation flags");
  if (!on) return;
  for (int q = 0; q < HDK_DEFL_MAX; ++q) D.h_ones[q].cond = q < D.k ? 1 : 0;
  cuda_check(cudaMemcpyAsync(D.ones, D.h_ones, HDK_DEFL_MAX * sizeof(hdk_pcg), cudaMemcpyHostToDevice, st_),
             "column deflation flags");
  const int cstride = static_cast<int>(sizeof(hdk_pcg) / sizeof(int));
  hdk_ok(hdk_scatter_cols(hf_.n, scene_.mesh.nv, HDK_DEFL_MAX, D.w, D.wv, df_.p2v, D.d, st_), "W by vertex");
  for (int g = 0; g < HDK_DEFL_MAX; g += 8)
    hdk_ok(hdk_bapply_cols_sorted(&dm_, dcomp_, D.wv + g * n3, n3, D.ef8 + g * 12 * ne, 12 * ne, corner_pos_,
                                  &D.ones[g].cond, cstride, 8, st_),
           "B W (columns)");
  hdk_ok(hdk_cpcg_apply_q(&dv_, &a_ff_, HDK_DEFL_MAX, D.ef8, 12 * ne, D.w, D.aw, D.ones, st_), "(A - B) W (columns)");
  hdk_ok(hdk_defl_gram(static_cast<int>(n3p), D.w, D.aw, D.part, D.ticket, D.d, st_), "E (columns)");
  kernel_launches += 5;
}

bool Engine::solve_columns_bcg(const ContactFrame& c, int r0, int& iterations) {
  ColumnSet& S = *cols_;
  if (!S.bst) build_columns_bcg();
  const int nv = scene_.mesh.nv, K = kColumns;
  const size_t n3 = 3 * static_cast<size_t>(nv);
  const int real = std::min(K, c.k - r0);
  for (int j = 0; j < K; ++j) {
    const int row = std::min(r0 + j, c.k - 1);
    hdk_ok(hdk_contact_column_init(&c.view, row, nv, df_.v2p, S.col[j].seed, S.col[j].x, st_), "column init");
  }
  *S.h_bm = real;
  cuda_check(cudaMemcpyAsync(S.bm, S.h_bm, sizeof(int), cudaMemcpyHostToDevice, st_), "block size");
  kernel_launches += K;
  if (ph_.on) cuda_check(cudaEventRecord(ph_.ev[6], st_), "phase event");
  LoopGraph& g = S.bgraph;
  if (g.exec) {
    cuda_check(cudaGraphLaunch(g.exec, st_), "columns (block CG)");
  } else {  // host-driven loop (profiling fallback)
    if (g.pre) cuda_check(cudaGraphLaunch(g.pre, st_), "columns (block CG)");
    for (;;) {
      cuda_check(cudaMemcpyAsync(S.h_any, S.any, sizeof(int), cudaMemcpyDeviceToHost, st_), "flag");
      cuda_check(cudaStreamSynchronize(st_), "sync");
      if (!*S.h_any) break;
      cuda_check(cudaGraphLaunch(g.body, st_), "columns (block CG)");
    }
  }
  cuda_check(cudaMemcpyAsync(S.h_bst, S.bst, sizeof(hdk_bcg), cudaMemcpyDeviceToHost, st_), "block CG state");
  cuda_check(cudaStreamSynchronize(st_), "columns (block CG) sync");
  const hdk_bcg& h = *S.h_bst;
  if (h.err == -1 || h.err == 10) {  // Gram matrix lost definiteness or the cap: column by column
    ++bcg_fallbacks;
    return false;
  }
  if (h.err != 0) raise(Code::AdjointDiverged, "backward step: contact column block CG failed");
  hdk_ok(hdk_cpcg_final(hf_.n, nv, K, S.xp_all, S.cz, S.x_all, df_.p2v, st_), "x = x + z (block)");
  cuda_check(cudaMemcpyAsync(cX_ + n3 * r0, S.x_all, n3 * real * sizeof(double), cudaMemcpyDeviceToDevice, st_),
             "columns");
  if (ph_.on) {
    cuda_check(cudaEventRecord(ph_.ev[7], st_), "phase event");
    cuda_check(cudaEventSynchronize(ph_.ev[7]), "phase event");
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ph_.ev[6], ph_.ev[7]) == cudaSuccess) ph_.col_ms += ms;
  }
  kernel_launches += g.counts[0] + static_cast<long long>(g.counts[1]) * h.iter + 1;
  const int per_col = 1 + h.iter;  // solves per column, as the column CG counts them
  ph_.col_batches += 1;
  ph_.col_iters += per_col;
  ph_.col_real_iters += static_cast<long long>(per_col) * real;
  column_solves += static_cast<long long>(per_col) * real;
  column_streams += per_col;
  iterations = per_col * real;
  return true;
}

bool Engine::solve_columns_pcg(const ContactFrame& c, int r0, int& iterations) {
  ColumnSet& S = *cols_;
  if (!S.cst) build_columns_pcg();
  const int nv = scene_.mesh.nv, K = kColumns;
  const size_t n3 = 3 * static_cast<size_t>(nv);
  for (int j = 0; j < K; ++j) {
    const int row = std::min(r0 + j, c.k - 1);
    hdk_ok(hdk_contact_column_init(&c.view, row, nv, df_.v2p, S.col[j].seed, S.col[j].x, st_), "column init");
  }
  kernel_launches += K;
  // profiling: per-chunk ring timestamps of this batch's multi-column passes
  // (HETERODYN_CHUNK_TRACE=path: the last traced batch is written at exit)
  static const char* trace_path = std::getenv("HETERODYN_CHUNK_TRACE");
  if (trace_path && !S.trace) {
    cuda_check(cudaMalloc(&S.trace, 4 * sizeof(long long) * df_.n_chunks), "chunk trace");
    cuda_check(cudaMallocHost(&S.h_trace_ptr, 2 * sizeof(long long*)), "chunk trace");
    S.h_trace_ptr[0] = S.trace;
    S.h_trace_ptr[1] = nullptr;
    S.trace_path = trace_path;
    S.trace_grid = df_.grid2;
    S.h_first2.resize(df_.grid2 + 1);
    cuda_check(cudaMemcpy(S.h_first2.data(), df_.first2, sizeof(int) * (df_.grid2 + 1), cudaMemcpyDeviceToHost),
               "first2");
    S.trace_chunks = df_.n_chunks;
  }
  static const char* cg_trace_path = std::getenv("HETERODYN_CG_TRACE");
  if (cg_trace_path && !S.cg_trace) {
    cuda_check(cudaMalloc(&S.cg_trace, sizeof(double) * K * 512 * 2), "cg trace");
    cuda_check(cudaMallocHost(&S.h_cg_trace_ptr, 2 * sizeof(double*)), "cg trace");
    S.h_cg_trace_ptr[0] = S.cg_trace;
    S.h_cg_trace_ptr[1] = nullptr;
    S.cg_trace_path = cg_trace_path;
  }
  if (S.cg_trace) {
    cuda_check(cudaMemsetAsync(S.cg_trace, 0, sizeof(double) * K * 512 * 2, st_), "cg trace");
    hdk_ok(hdk_set_cpcg_trace(S.h_cg_trace_ptr, st_), "cg trace");
  }
  if (S.trace) {
    cuda_check(cudaMemsetAsync(S.trace, 0, 4 * sizeof(long long) * df_.n_chunks, st_), "chunk trace");
    hdk_ok(hdk_set_chunk_trace(S.h_trace_ptr, st_), "chunk trace");
  }
  if (ph_.on) cuda_check(cudaEventRecord(ph_.ev[6], st_), "phase event");
  LoopGraph& g = S.pgraph;
  if (g.exec) {
    cuda_check(cudaGraphLaunch(g.exec, st_), "columns (CG)");
  } else {  // host-driven loop (profiling fallback)
    if (g.pre) cuda_check(cudaGraphLaunch(g.pre, st_), "columns (CG)");
    for (;;) {
      cuda_check(cudaMemcpyAsync(S.h_any, S.any, sizeof(int), cudaMemcpyDeviceToHost, st_), "flag");
      cuda_check(cudaStreamSynchronize(st_), "sync");
      if (!*S.h_any) break;
      cuda_check(cudaGraphLaunch(g.body, st_), "columns (CG)");
    }
  }
  if (S.trace) hdk_ok(hdk_set_chunk_trace(S.h_trace_ptr + 1, st_), "chunk trace off");
  cuda_check(cudaMemcpyAsync(S.h_cst, S.cst, sizeof(hdk_pcg) * K, cudaMemcpyDeviceToHost, st_), "pcg state");
  cuda_check(cudaStreamSynchronize(st_), "columns (CG) sync");
  const int real = std::min(K, c.k - r0);
  int iters = 0, most = 0;
  for (int j = 0; j < real; ++j) {
    const hdk_pcg& h = S.h_cst[j];
    if (h.err == -1) {  // not positive definite along a direction: Anderson for this batch
      ++pcg_fallbacks;
      return false;
    }
    if (h.err != 0) raise(Code::AdjointDiverged, "backward step: contact column CG did not settle (cap or non-finite values)");
    iters += 1 + h.iter;
    most = std::max(most, h.iter);
  }
  for (int j = real; j < K; ++j) most = std::max(most, S.h_cst[j].iter);
  hdk_ok(hdk_cpcg_final(hf_.n, nv, K, S.xp_all, S.cz, S.x_all, df_.p2v, st_), "x = x + z (columns)");
  cuda_check(cudaMemcpyAsync(cX_ + n3 * r0, S.x_all, n3 * real * sizeof(double), cudaMemcpyDeviceToDevice, st_),
             "columns");
  if (ph_.on) {
    cuda_check(cudaEventRecord(ph_.ev[7], st_), "phase event");
    cuda_check(cudaEventSynchronize(ph_.ev[7]), "phase event");
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ph_.ev[6], ph_.ev[7]) == cudaSuccess) ph_.col_ms += ms;
  }
  kernel_launches += g.counts[0] + static_cast<long long>(g.counts[1]) * most + 1;
  ph_.col_batches += 1;
  ph_.col_iters += 1 + most;
  ph_.col_real_iters += iters;
  column_solves += iters;
  column_streams += 1 + most;
  iterations = iters;
  return true;
}

int Engine::solve_columns(const ContactFrame& c, int r0) {
  if (!cols_) build_columns();
  if (use_pcg_) {
    static const bool block = [] {  // HETERODYN_COLUMN_CG=column: one CG per column (A/B)
      const char* e = std::getenv("HETERODYN_COLUMN_CG");
      return !(e && std::string(e) == "column");
    }();
    int it = 0;
    if (block && c.k - r0 > 1 && solve_columns_bcg(c, r0, it)) return it;
    if (solve_columns_pcg(c, r0, it)) return it;
  }
  ColumnSet& S = *cols_;
  const int nv = scene_.mesh.nv;
  for (int j = 0; j < kColumns; ++j) {
    const int row = std::min(r0 + j, c.k - 1);
    hdk_ok(hdk_contact_column_init(&c.view, row, nv, df_.v2p, S.col[j].seed, S.col[j].x, st_), "column init");
  }
  kernel_launches += kColumns;
  if (ph_.on) cuda_check(cudaEventRecord(ph_.ev[6], st_), "phase event");
  if (S.graph.exec) {
    cuda_check(cudaGraphLaunch(S.graph.exec, st_), "columns");
  } else {  // host-driven loop (profiling fallback)
    if (S.graph.pre) cuda_check(cudaGraphLaunch(S.graph.pre, st_), "columns");
    for (;;) {
      cuda_check(cudaGraphLaunch(S.graph.body, st_), "columns");
      cuda_check(cudaMemcpyAsync(S.h_any, S.any, sizeof(int), cudaMemcpyDeviceToHost, st_), "flag");
      cuda_check(cudaStreamSynchronize(st_), "sync");
      if (!*S.h_any) break;
    }
  }
  if (ph_.on) cuda_check(cudaEventRecord(ph_.ev[7], st_), "phase event");
  cuda_check(cudaMemcpyAsync(S.h_ctls, S.ctls, sizeof(hdk_ctl) * kColumns, cudaMemcpyDeviceToHost, st_), "ctl read");
  cuda_check(cudaStreamSynchronize(st_), "columns sync");
  if (ph_.on) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ph_.ev[6], ph_.ev[7]) == cudaSuccess) ph_.col_ms += ms;
  }
  int iters = 0, most = 0;
  const size_t n3 = 3 * static_cast<size_t>(nv);
  for (int j = 0; j < kColumns && r0 + j < c.k; ++j) {
    hdk_ctl& h = S.h_ctls[j];
    if (h.err == 0 && h.nonfinite) h.err = 10;
    if (h.err != 0) {
      std::memcpy(h_ctl_, &h, sizeof(hdk_ctl));
      check_ctl("backward step (contact column)");
    }
    iters += h.iterations;
    most = std::max(most, h.iterations);
    cuda_check(cudaMemcpyAsync(cX_ + n3 * (r0 + j), S.col[j].x, n3 * sizeof(double), cudaMemcpyDeviceToDevice, st_),
               "column");
  }
  kernel_launches += S.graph.counts[0] + static_cast<long long>(S.graph.counts[1]) * ((most + unroll_ - 1) / unroll_);
  ph_.col_batches += 1;
  ph_.col_iters += most;
  column_solves += iters;
  column_streams += most;
  ph_.col_real_iters += iters;
  return iters;
}

}  // namespace hdb
