// Batched system-ID evaluation: one GPU's
// share of a batch of material-parameter samples.  Default (lockstep): all
// samples are one segmented engine (engine_seg.cpp) — concatenated index
// spaces, one block-diagonal factor stream, per-sample loop control — so
// every kernel processes all of the GPU's samples in one launch.  Scenes the
// segmented engine does not take (contact, Dirichlet vertices, hooks) and
// HETERODYN_BATCH=streams use one engine per sample on its own CUDA stream,
// driven concurrently by host worker threads.  One evaluation is
// the reference's identify objective for every sample (run_identify,
// drivers.cpp:848-851; roll + chain_backward, drivers.cpp:31-99):
//   L_s = 1/2 |q_T(E_s) - q_target|^2,  dL_s/dE_s  (per element)
// and the fixed-order sum over the local samples of [L_s, dL_s/dE] lands in
// one device vector — the only data that crosses GPUs (NCCL all-reduce).
#pragma once

#include <memory>
#include <vector>

#include "engine.hpp"

namespace hdb {

class Batch {
 public:
  Batch(const Scene& scene, int samples, const double* young, int threads, int solve_ctas = 0);
  ~Batch();
  Batch(const Batch&) = delete;
  Batch& operator=(const Batch&) = delete;

  int samples() const { return samples_; }
  void set_target(const double* q_target);
  // New per-sample Young's moduli (samples x element_count): every sample
  // refactors (Engine::set_young), in parallel over the host threads.
  void set_young(const double* young, bool freeze_means);
  // Runs every sample's trajectory + adjoint; loss (samples) and grad_sum
  // (element_count) are host outputs and may be null; device_out (1 +
  // element_count doubles on this device) receives [sum L, sum dL/dE].
  void evaluate(int frames, double* loss, double* grad_sum, double* device_out);
  long long kernel_launches() const;
  // ms per solve (reps after warm-up) of the batch's solve path: the lockstep
  // engine's block-diagonal factor (every sample in one launch per pass), or
  // sample 0's factor; *bytes: that solve's algorithmic bytes
  double time_solve(int reps, double* bytes);
  void evaluate_lockstep(int frames, double* loss, double* grad_sum, double* device_out);
  long long solve_count() const;      // 3-axis global solves over all samples so far
  double solve_bytes() const;         // algorithmic bytes of one solve of one sample (16 nnz(S') + 96 n)
  cudaStream_t stream() const { return st_; }
  bool lockstep() const { return lock_ != nullptr; }
  // lockstep: sum over samples of their own (fwd + adjoint) iteration counts
  long long sample_iterations() const { return lock_ ? lock_->seg_sample_iterations : solve_count(); }
  double last_ms = 0;  // device-side duration of the last evaluate (max over sample streams)

 private:
  const Scene& scene_;
  std::vector<std::unique_ptr<Engine>> eng_;
  std::unique_ptr<Scene> seg_scene_;  // lockstep: the concatenated scene (outlives lock_)
  std::unique_ptr<Engine> lock_;
  int samples_ = 0;
  int threads_ = 1, device_ = 0;
  cudaStream_t st_ = nullptr;
  double* target_ = nullptr;   // 3 nv
  double* loss_ = nullptr;     // samples
  double* out_ = nullptr;      // 1 + ne
  const double** grads_ = nullptr;  // samples device pointers
  long long own_launches_ = 0;
};

}  // namespace hdb
