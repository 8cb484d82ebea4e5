// Device-resident forward/backward PD engine (one hd_sim).  The reference's
// forward_step (forward.cpp:148-272), backward_step (backward.cpp:396-414),
// roll/chain_backward (drivers.cpp:31-99) and GlobalSystem (factor.hpp:85-130)
// re-designed for sm_100a: all per-iteration state stays in HBM, the PD and
// adjoint fixed-point loops run inside CUDA graphs whose WHILE conditional
// node is driven by the device-side dual gate, and only per-step status
// crosses back to the host.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/hdk.h"
#include "host.hpp"

namespace hdb {

struct DevArena {
  std::vector<void*> ptrs;
  ~DevArena();
  void* raw(size_t bytes);
  template <class T>
  T* alloc(size_t n) { return static_cast<T*>(raw(sizeof(T) * (n ? n : 1))); }
  template <class T>
  T* upload(const std::vector<T>& v) {
    T* p = alloc<T>(v.size());
    if (!v.empty()) copy_h2d(p, v.data(), sizeof(T) * v.size());
    return p;
  }
  static void copy_h2d(void* d, const void* h, size_t bytes);
};

void cuda_check(cudaError_t e, const char* what);
// Zero device memory and wait for it: a plain cudaMemset runs on the legacy
// stream, which does not order against the engines' non-blocking streams, so
// a buffer zeroed after the engine started (lazily built graphs) could be
// cleared while its first kernels already run (seen as nondeterminism with
// several engines per process, HETERODYN_BATCH=streams).
void cuda_zero(void* p, size_t bytes, const char* what);

struct LoopGraph {
  cudaGraphExec_t exec = nullptr, pre = nullptr, body = nullptr, post = nullptr;
  int counts[3] = {0, 0, 0};
  void destroy() {
    for (cudaGraphExec_t* e : {&exec, &pre, &body, &post})
      if (*e) {
        cudaGraphExecDestroy(*e);
        *e = nullptr;
      }
  }
};


// pre -> while(body) -> post as one executable graph with a device-driven
// WHILE conditional node (engine.cpp).
void build_loop_graph(cudaStream_t st, bool use_cond, const std::function<void()>& pre,
                      const std::function<void(unsigned long long)>& body, const std::function<void()>& post,
                      LoopGraph& out);

// A contact set in device memory: one allocation carved by
// hdk_contact_block_layout (capacities, counts, rows, inverse columns, W,
// multipliers, weights).  The engine's working set is one; every recorded
// frame with contacts keeps a copy for the adjoint (same capacities, one D2D
// copy).  nc/nf/k/nu are host copies of the device counts, valid after the
// step's status read.
struct ContactFrame {
  int nc = 0, nf = 0, k = 0, nu = 0;
  void* base = nullptr;
  size_t bytes = 0;
  hdk_contacts view{};
  ContactFrame() = default;
  ContactFrame(const ContactFrame&) = delete;
  ContactFrame& operator=(const ContactFrame&) = delete;
  ~ContactFrame();
  void allocate(int cap_c, int cap_k, int cap_u, int n);  // (re)allocates when the layout differs
};

// pre -> [while] -> ... as one executable graph: segments in order, a loop
// segment is a WHILE conditional node whose body the segment's function
// captures (it receives the node's handle and sets the condition on the
// device).  Without conditional nodes (HETERODYN_NO_COND_GRAPH=1) every
// segment is its own executable and the host drives the loops from `flag`.
struct SeqGraph {
  struct Seg {
    bool loop = false;
    bool check_first = false;     // loop condition set before the node (else it starts at 1)
    const int* flag = nullptr;    // device word holding the loop condition (host-driven mode)
    std::function<void(unsigned long long)> fn;
  };
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaGraphExec_t> parts;
  std::vector<Seg> segs;
  std::vector<int> kernels;  // kernel nodes per segment
  void destroy() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    for (cudaGraphExec_t e : parts)
      if (e) cudaGraphExecDestroy(e);
    parts.clear();
  }
};
void build_seq_graph(cudaStream_t st, bool use_cond, std::vector<SeqGraph::Seg> segs, SeqGraph& out);

struct GradOut {
  Vec dl_dq0, dl_dv0, dl_df_ext, dl_de, dl_dw;
  std::vector<double> tau, rho;
  int adjoint_iterations = 0;
};

class Engine {
 public:
  // Turns recycled-subspace deflation of the backbone CG on or off for the
  // following solves and drops the recycled subspace (engine_pcg.cpp).
  void set_deflation(bool on);
  // The fp32 copy of the factor values (the adjoint CG's preconditioner), re-made after every S' build.
  void refresh_fp32();
  // young: optional per-element Young's moduli replacing the scene's (a
  // parameter sample of a batch); the factor is built once for them.
  // solve_ctas: cap on the CTAs of each solve pass (0 = one resident wave).
  // shared_device: other engines run concurrently on the device (a batch's
  // samples): the backbone then stays on one stream.
  // segments > 1: `scene` is a lockstep batch of that many copies of one mesh
  // (make_segmented_scene): one block-diagonal factor, per-sample loop
  // control (hdk_seg_*), every sample stopping at its own iteration count.
  explicit Engine(const Scene& scene, const Vec* young = nullptr, int solve_ctas = 0, bool shared_device = false,
                  int segments = 1);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  void step();  // throws Error; state untouched on failure
  void record(bool on);
  void reserve_frames(int frames);  // allocate recorded-frame slots ahead of time
  int recorded() const { return nrec_; }
  // keep_frames: recorded frames stay valid (the C++ solver API sets the
  // state of every step from the caller's SimState)
  void set_state(const double* q, const double* v, double time, bool keep_frames = false);
  // One forward step recorded into frame slot `slot` (allocated on demand)
  // instead of the append position: the C++ solver API's ForwardCache owns a
  // slot until it is destroyed (solver_api.cpp).
  void step_into(int slot);
  // backward_step (backward.cpp:396-414) for the frame in `slot` alone, seeded
  // with dL/dq_{t+1}, dL/dv_{t+1} (host, NULL = zero); GradOut holds the step's
  // input gradients (dl_dq0/dl_dv0 = dL/dq_t, dL/dv_t), tau/rho one entry.
  GradOut backward_slot(int slot, const double* dl_dq_next, const double* dl_dv_next);
  // trust-region band of the adjoint (SolverConfig::eps_tr); re-captures the
  // backward graphs when it changes
  void set_eps_tr(double eps_tr);
  double eps_tr() const { return eps_tr_; }
  int slot_count() const { return static_cast<int>(slots_.size()); }
  // host copy of a recorded frame's q~ (which = 0) or next-to-last iterate (1)
  Vec frame_vector(int slot, int which) const;
  void set_external_force(const double* f);  // dof doubles into the device f_ext the graphs read
  void external_force_into(double* out) const;
  double last_fb_residual() const;  // max |FB residual| over the last step's normal contacts
  // Contact rows (vertex, obstacle) of the last step and its per-iteration
  // clamp / cone decision values ([iteration][nc], [iteration][nf], hdk_contact_trace).
  void contact_trace(std::vector<int>& vertex, std::vector<int>& obstacle, std::vector<double>& clamp,
                     std::vector<double>& cone, int& nc, int& nf, int& iterations) const;
  double penetration() const;       // deepest obstacle penetration of the current state
  // canonical: seed from device state, L = 1/2|q_T - ref|^2 (+ 1/2|v_T|^2 when
  // d_target is null and ref is the rest shape); d_target is a device array.
  // sinks: host buffers (any may be NULL) the gradients are copied into
  // directly, with one stream synchronisation; without sinks and with
  // download, GradOut's vectors are filled instead.
  struct GradSinks {
    double *dq0 = nullptr, *dv0 = nullptr, *df_ext = nullptr, *de = nullptr, *dw = nullptr;
  };
  GradOut backward(const double* dl_dq_direct, const double* dl_dq_final, const double* dl_dv_final,
                   bool canonical = false, bool download = true, const double* d_target = nullptr,
                   const GradSinks* sinks = nullptr);
  size_t dw_count() const;  // entries of dL/dw (2 n_e corotated, n_e Neo-Hookean)
  void reset_state();  // scene's initial state, time 0, recorded frames dropped
  double time_solve(int reps, double* bytes);
  double time_backbone(int reps, unsigned skip_mask);
  void backbone_body(unsigned long long cond_handle, unsigned skip_mask);
  // Profiling (HETERODYN_PHASES=1): CUDA-event time per step phase, summed
  // and printed to stderr when the engine is destroyed.
  struct Phases {
    bool on = false;
    bool skip_first = true;
    cudaEvent_t ev[8] = {};
    double ms[8] = {};
    long long n = 0;
    double col_ms = 0;  // contact columns: time, batches, batched and per-column iterations
    long long col_batches = 0, col_iters = 0, col_real_iters = 0;
    bool per_frame = false;  // HETERODYN_PHASES=2: one stderr line per backward frame
    double last_col_ms = 0;
  } ph_;
  void phase_mark(int i);
  void phase_collect(int first, int last);
  void trace_backbone(int reps, std::vector<double>& out);
  // Contact adjoint columns x_c = (A - B)^{-1} j_c (backward.cpp:229-238),
  // kColumns at a time: one multi-column stream of the factor per iteration,
  // each column's Anderson kernels on its own pair of streams
  // (engine_columns.cpp).
  static constexpr int kColumns = HDK_BB_COLUMNS;
  struct ColumnSet;
  struct ColumnSetDeleter {
    void operator()(ColumnSet* p) const;  // engine_columns.cpp
  };
  std::unique_ptr<ColumnSet, ColumnSetDeleter> cols_;
  void build_columns();
  // Solves rows [r0, r0 + kColumns) of contact frame c (rows past k repeat
  // the last one); returns the iterations of the real columns.
  int solve_columns(const ContactFrame& c, int r0);
  // The same rows by column-batched CG (the default with use_pcg_); false
  // when a column's p.q <= 0 (the caller runs the Anderson columns).
  bool solve_columns_pcg(const ContactFrame& c, int r0, int& iterations);
  void build_columns_pcg();
  // The same rows by block CG over the batch (the default; a batch of one row
  // and a lost-definiteness / cap failure go to solve_columns_pcg).
  bool solve_columns_bcg(const ContactFrame& c, int r0, int& iterations);
  void column_deflation_setup();
  void build_columns_bcg();
  // All K columns of contact frame c through the kColumns slots, a finished
  // slot refilled with the next row (the loop exits when a column finishes);
  // returns the columns' iterations.  Opt-in (HETERODYN_COLUMN_REFILL=1): the
  // per-refill host round trip cost more than the idle slots it saved; the
  // default is batches of kColumns rows (solve_columns).
  int solve_all_columns(const ContactFrame& c);
  void column_pre(int slot);
  void columns_body(unsigned long long cond_handle, unsigned skip);
  double time_columns(int reps, unsigned skip);  // profiling: ms per multi-column iteration
  void trace_loop(std::vector<double>& out);
  unsigned long long* loop_trace_ = nullptr;  // set only while trace_loop runs
  int last_backward_iterations_ = 0;
  Vec solve_free(const double* rhs, const double* fixed_q);
  void set_young(const Vec& young, bool freeze);
  // Device refactorization (engine_refactor.cpp, refactor.cu): the numeric
  // part of a same-pattern set_young on the GPU.  Plans are built on first use.
  struct DeviceRefactor;
  struct DeviceRefactorDeleter {
    void operator()(DeviceRefactor* p) const;
  };
  std::unique_ptr<DeviceRefactor, DeviceRefactorDeleter> drf_;
  bool refactor_on_device();  // false: this factor cannot (host path)
  void refactor_device_values();
  double last_refactor_ms = 0;  // host wall time of the last set_young
  bool last_refactor_device = false;

  Vec positions() const;
  Vec velocities() const;
  // the same straight into a host buffer of 3 n_v doubles (one stream sync)
  void positions_into(double* host) const;
  void velocities_into(double* host) const;
  size_t dof_count() const { return 3 * static_cast<size_t>(scene_.mesh.nv); }
  double time() const { return time_; }
  int dofs() const { return 3 * mesh().nv; }
  int last_iterations = 0, last_converged = 0, last_contacts = 0;
  int segments() const { return segs_; }
  const hdk_segs& segs() const { return dseg_; }
  std::vector<int> seg_iterations;   // segmented batch: forward iterations of the last step, per sample
  std::vector<int> seg_converged;
  std::vector<double> seg_tau;       // segmented batch: tau of the last backward frame, per sample
  long long seg_sample_iterations = 0;  // sum over samples of their own iteration counts (fwd solves + adjoint)
  long long solve_count = 0, a_spmv_count = 0, refactor_count = 0, kernel_launches = 0;
  // Contact-adjoint column solves (inside solve_count) and the multi-column
  // factor streams that carried them (kColumns columns per stream).
  long long column_solves = 0, column_streams = 0;
  long long factor_streams() const { return solve_count - column_solves + column_streams; }
  const HostFactor& factor() const { return hf_; }
  const Mesh& mesh() const { return scene_.mesh; }
  const Material& material() const { return mat_; }
  cudaStream_t stream() const { return st_; }
  const double* d_positions() const { return q_; }
  const double* d_dl_de() const { return dle_; }

 private:
  struct Frame;
  void add_slot();
  void build_static();
  void build_factor_device();
  void upload_material();                 // material arrays + scalars into the existing buffers
  void fill_factor_values(double* sval);  // hf_'s S' values into a stream buffer
  void build_forward_graph();
  void build_backward_graph();
  void run_graph(LoopGraph& g, const char* what);
  void backward_frame(int t, GradOut& out);
  // segmented batch (engine_seg.cpp)
  void build_forward_graph_seg();
  void build_backward_graph_seg();
  void backbone_body_seg(unsigned long long cond_handle);
  // adjoint backbone by preconditioned CG (pcg.cu, engine_pcg.cpp), the
  // default for a single problem (HETERODYN_ADJOINT=aa: the reference's
  // Anderson loop); falls back to the Anderson loop when A - B is not
  // positive definite along a search direction
  bool use_pcg_ = true;
  std::unique_ptr<LoopGraph> pgraph_;
  hdk_pcg* pcg_ = nullptr;
  hdk_pcg* h_pcg_ = nullptr;
  double *pcg_part_ = nullptr, *pr_ = nullptr, *pz_ = nullptr, *pp_ = nullptr, *pq_ = nullptr, *pap_ = nullptr,
         *prp_ = nullptr, *ppv_ = nullptr;
  unsigned int* pcg_ticket_ = nullptr;
  // Deflated backbone CG (engine_pcg.cpp, pcg.cu hdk_defl): Ritz vectors of a
  // recorded backbone CG, recycled across steps.
  struct Deflation {
    bool on = false;        // HETERODYN_DEFLATION != 0 and a single (non-segmented) engine
    bool valid = false;     // W holds Ritz vectors
    int k = 0, hcap = 0, plain_iters = 0;
    int misses = 0, cooldown = 0;  // deflated solves that did not pay; plain solves left before retrying
    hdk_defl* d = nullptr;  // device state
    hdk_defl* h = nullptr;  // pinned mirror (the int fields are uploaded per solve)
    hdk_pcg* ones = nullptr;  // run flags of the 8-column B apply / q kernels
    hdk_pcg* h_ones = nullptr;
    double *w = nullptr, *aw = nullptr, *wv = nullptr, *ef8 = nullptr, *zhist = nullptr, *hist = nullptr,
           *coef = nullptr, *part = nullptr, *h_hist = nullptr, *h_coef = nullptr;
    unsigned int* ticket = nullptr;
    long long refreshes = 0, deflated_solves = 0;
    // lockstep batch (per sample): E factors / coefficients, E scratch, per-sample tickets
    hdk_sdefl* ds = nullptr;
    double* e = nullptr;
    unsigned int* tickets = nullptr;
  } defl_;
  void defl_after_solve_seg();
  void defl_alloc();

  void defl_after_solve(int iterations, bool converged);
  long long pcg_fallbacks = 0, bcg_fallbacks = 0;
  void build_pcg_graph();
  void build_pcg_graph_seg();
  bool run_pcg(int& iterations);  // false: fall back to the Anderson backbone
  bool host_any() const;
  void load_frame(int t);  // frame slot t into the backward working buffers
  void sync_ctl();
  void check_ctl(const char* what);

  const Scene& scene_;
  Material mat_;
  HostFactor hf_;
  cudaStream_t st_ = nullptr;
  cudaStream_t st2_ = nullptr;  // second branch of the backbone graph (coefficient solve)
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  std::unique_ptr<DevArena> mem_;      // mesh/material/state/work
  std::unique_ptr<DevArena> fmem_;     // factor (rebuilt on refresh)
  bool use_cond_ = true;
  int solve_ctas_ = 0;
  double time_ = 0;

  // device views
  hdk_mesh dm_{};
  hdk_material dmat_{};
  hdk_factor df_{};
  hdk_vtx dv_{};
  hdk_csr a_ff_{}, a_fd_{}, a_df_{};
  int* d_fixed_ = nullptr;

  // state / work buffers (3 nv doubles unless noted)
  double *q_ = nullptr, *v_ = nullptr, *fext_ = nullptr;
  double *qtil_ = nullptr, *qcur_ = nullptr, *qprev_ = nullptr, *qhat_ = nullptr, *bprev_ = nullptr, *damp_ = nullptr;
  double *rhs_ = nullptr, *fixc_ = nullptr;  // 3 n
  double *ef_ = nullptr, *ef2_ = nullptr;    // 12 ne
  double *lastq_ = nullptr, *lastg_ = nullptr, *dq_ = nullptr, *dg_ = nullptr;  // dq/dg: 8 x 3 nv
  double *part_a_ = nullptr, *part_b_ = nullptr, *part_c_ = nullptr;
  double* cache_ = nullptr;  // 24 ne projection cache of the current step
  hdk_ctl* ctl_ = nullptr;
  unsigned int* ticket_ = nullptr;
  hdk_ctl* snap_ = nullptr;  // control-block snapshot of the backbone (hdk_bb_dots -> hdk_bb_mix)
  int unroll_ = 4;           // backbone iterations per WHILE-loop body
  bool branch_ = true;       // coefficient solve on its own graph branch (st2_)
  bool device_values_ = true;  // factor values built on the device (inverse.cu)
  std::vector<int> order_cache_;  // fill-reducing ordering, reused by every refactorization
  double* seedp_ = nullptr;  // adjoint seed in elimination order (3 n)
  double* xp_ = nullptr;     // backbone iterate in elimination order (3 n); x_ holds it by vertex
  int* corner_pos_ = nullptr;  // element corner -> slot in the elimination-order incidence list
  int* corner_vpos_ = nullptr;  // element corner -> slot in the vertex-ordered incidence list
  // R = gather o B in elimination order: R(t), tracked R(x), last R(x) and R(g), R(dq_j + dg_j) ring
  double *rt_ = nullptr, *rx_ = nullptr, *lrx_ = nullptr, *lrg_ = nullptr, *rsq_ = nullptr;
  double* tv_ = nullptr;     // t by vertex (input of B t)
  void* aares_ = nullptr;    // coefficient-solve result (hdk_bb_solve -> hdk_bb_mix)  // last-block ticket of hdk_aa_dots_fused
  hdk_ctl* h_ctl_ = nullptr;  // pinned mirror
  double* h_stage_ = nullptr;  // pinned material staging (upload_material), 6 n_e doubles
  double* hook_ = nullptr;    // 5 doubles device

  // backward work
  double *seed_ = nullptr, *x_ = nullptr, *t_ = nullptr, *mu_ = nullptr, *bmu_ = nullptr, *dcomp_ = nullptr;
  double *qbar_ = nullptr, *vbar_ = nullptr, *dlq_ = nullptr, *dlv_ = nullptr, *dfacc_ = nullptr, *coup_ = nullptr;
  double *dlw_ = nullptr, *dle_ = nullptr, *eprev_ = nullptr, *estar_ = nullptr, *dqp_ = nullptr, *direct_ = nullptr;
  // working copy of one recorded frame for the backward graph
  double *bq_t_ = nullptr, *bv_t_ = nullptr, *bqtil_ = nullptr, *bqprev_ = nullptr, *bqstar_ = nullptr, *bcache_ = nullptr;

  struct Frame {
    double *q_t, *v_t, *qtil, *qprev, *qstar, *cache;
    std::shared_ptr<ContactFrame> contacts;  // reused across recordings
    bool has_contacts = false;
  };
  std::vector<Frame> slots_;  // device storage of recorded frames (reused)
  std::vector<std::unique_ptr<DevArena>> frame_mem_;
  int nrec_ = 0;
  bool recording_ = false;
  int force_slot_ = -1;  // step_into: the slot this step records into
  int segs_ = 1;         // samples of a lockstep batch (1: a single problem)
  hdk_segs dseg_{};
  int* any_ = nullptr;                // OR over the samples' loop conditions
  unsigned int* gate_ticket_ = nullptr;
  double* part18_ = nullptr;          // quantity-major Anderson partials (zero-initialised)
  int* seg_windows_ = nullptr;        // per-sample Anderson window (forward)
  double* seg_means_dev_ = nullptr;   // per-sample prox means
  double eps_tr_ = 0.1;
  int aa_window_ = 1;

  double* rest_ = nullptr;  // rest positions (canonical loss seed)
  int fk_pre_ = 0, fk_body_ = 0, fk_post_ = 0, bk_pre_ = 0, bk_body_ = 0, bk_post_ = 0;
  std::unique_ptr<LoopGraph> fgraph_, bgraph_;
  cudaGraphExec_t bpre_ = nullptr, bpost_a_ = nullptr, bpost_b_ = nullptr;
  // contact: working set of the current step, its trace and scratch
  double* obst_ = nullptr;  // HDK_OBSTACLE_DOUBLES per obstacle
  double* q0c_ = nullptr;   // contact-free solve result of one iteration (full)
  ContactFrame cw_;
  int* h_cnt_ = nullptr;    // pinned mirror of cw_.view.cnt
  double* cM_ = nullptr;    // global scratch of the dense systems when they exceed shared memory
  size_t cM_len_ = 0;
  hdk_contact_trace ctr_{};
  void* ctr_mem_ = nullptr;
  int trace_iters_ = 0;     // iterations recorded in ctr_ by the last step
  double *cX_ = nullptr, *cz0_ = nullptr;
  size_t cX_cols_ = 0;
  SeqGraph cgraph_;         // forward graph of scenes with obstacles
  int fc_kernels_[5] = {0, 0, 0, 0, 0};
  void ensure_contact_capacity(int need_c, int need_k, int need_u);
  void build_contact_graph();
  bool run_contact_step();  // false: capacities grown, step must be re-run
  bool cur_has_contacts_ = false;
};

}  // namespace hdb
