// Batched system-ID evaluation; see batch.hpp.
#include "batch.hpp"

#include <algorithm>
#include <cstdlib>
#include <string>
#include <atomic>
#include <exception>
#include <mutex>
#include <thread>

namespace hdb {

namespace {

void hdk_check_b(int status, const char* what) {
  if (status != 0) raise(Code::InvalidArgument, std::string("CUDA launch failed: ") + what);
}

// Runs body(i) for i in [0, count) on `threads` host threads (static
// round-robin: sample i goes to thread i % threads, so a sample's work is
// always issued from the same thread); the first exception is rethrown.
template <class F>
void parallel_samples(int count, int threads, int device, F&& body) {
  std::exception_ptr err;
  std::mutex m;
  const auto run = [&](int t) {
    int cur = -1;
    try {
      cuda_check(cudaSetDevice(device), "set device");
      for (int i = t; i < count; i += threads) {
        cur = i;
        body(i);
      }
    } catch (const Error& e) {
      std::lock_guard<std::mutex> g(m);
      if (!err) err = std::make_exception_ptr(Error(e.code, "sample " + std::to_string(cur) + ": " + e.what()));
    } catch (...) {
      std::lock_guard<std::mutex> g(m);
      if (!err) err = std::current_exception();
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(run, t);
  run(0);
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace

Batch::Batch(const Scene& scene, int samples, const double* young, int threads, int solve_ctas) : scene_(scene) {
  if (samples < 1) raise(Code::InvalidArgument, "hd_batch_create: at least one sample required");
  if (!scene.obstacles.empty())
    raise(Code::InvalidArgument, "hd_batch_create: batched system-ID runs contact-free scenes (config C5)");
  cuda_check(cudaGetDevice(&device_), "get device");
  samples_ = samples;
  const char* mode = std::getenv("HETERODYN_BATCH");
  const bool streams = (mode && std::string(mode) == "streams") || !scene.fixed.empty() || scene.hook;
  if (!streams) {  // all samples in one segmented engine
    seg_scene_ = std::make_unique<Scene>(make_segmented_scene(scene, samples, young));
    lock_ = std::make_unique<Engine>(*seg_scene_, nullptr, solve_ctas, false, samples);
    st_ = lock_->stream();
    const size_t n3 = 3 * static_cast<size_t>(scene.mesh.nv) * samples;
    cuda_check(cudaMalloc(&target_, n3 * sizeof(double)), "target");
    cuda_check(cudaMemcpy(target_, seg_scene_->q0.data(), n3 * sizeof(double), cudaMemcpyHostToDevice), "target");
    cuda_check(cudaMalloc(&loss_, samples * sizeof(double)), "loss");
    cuda_check(cudaMalloc(&out_, (1 + static_cast<size_t>(scene.mesh.ne)) * sizeof(double)), "out");
    return;
  }
  threads_ = std::max(1, std::min(threads, samples));
  // Several samples' solves share the SMs: cap each pass at a quarter wave
  // (measured on C5: 975 ms -> 778 ms per 64 x 10-frame evaluation).
  if (solve_ctas == 0 && samples >= 4) solve_ctas = 37;
  const int ne = scene.mesh.ne;
  eng_.resize(samples);
  parallel_samples(samples, threads_, device_, [&](int s) {
    if (young) {
      Vec y(young + static_cast<size_t>(s) * ne, young + static_cast<size_t>(s + 1) * ne);
      eng_[s] = std::make_unique<Engine>(scene, &y, solve_ctas, true);
    } else {
      eng_[s] = std::make_unique<Engine>(scene, nullptr, solve_ctas, true);
    }
  });
  cuda_check(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "batch stream");
  const size_t n3 = 3 * static_cast<size_t>(scene.mesh.nv);
  cuda_check(cudaMalloc(&target_, n3 * sizeof(double)), "target");
  cuda_check(cudaMemcpy(target_, scene.q0.data(), n3 * sizeof(double), cudaMemcpyHostToDevice), "target");
  cuda_check(cudaMalloc(&loss_, samples * sizeof(double)), "loss");
  cuda_check(cudaMalloc(&out_, (1 + static_cast<size_t>(ne)) * sizeof(double)), "out");
  std::vector<const double*> g(samples);
  for (int s = 0; s < samples; ++s) g[s] = eng_[s]->d_dl_de();
  cuda_check(cudaMalloc(&grads_, samples * sizeof(double*)), "grad pointers");
  cuda_check(cudaMemcpy(grads_, g.data(), samples * sizeof(double*), cudaMemcpyHostToDevice), "grad pointers");
}

Batch::~Batch() {
  eng_.clear();
  for (void* p : {static_cast<void*>(target_), static_cast<void*>(loss_), static_cast<void*>(out_),
                  static_cast<void*>(grads_)})
    if (p) cudaFree(p);
  if (st_ && !lock_) cudaStreamDestroy(st_);  // lockstep: the engine's stream
  lock_.reset();
}

void Batch::set_target(const double* q) {
  const size_t n3 = 3 * static_cast<size_t>(scene_.mesh.nv);
  const int copies = lock_ ? samples_ : 1;  // lockstep: one copy per sample
  for (int k = 0; k < copies; ++k)
    cuda_check(cudaMemcpy(target_ + k * n3, q, n3 * sizeof(double), cudaMemcpyHostToDevice), "target");
}

void Batch::evaluate(int frames, double* loss, double* grad_sum, double* device_out) {
  if (frames < 1) raise(Code::InvalidArgument, "hd_batch_evaluate: frames must be >= 1");
  if (lock_) {
    evaluate_lockstep(frames, loss, grad_sum, device_out);
    return;
  }
  const int S = samples(), ne = scene_.mesh.ne;
  const int n3 = 3 * scene_.mesh.nv;
  // frame slots are allocated up front, never while other samples' graphs run
  parallel_samples(S, threads_, device_, [&](int s) { eng_[s]->reserve_frames(frames); });
  struct Events {  // destroyed on every exit path (a failing sample rethrows)
    cudaEvent_t start = nullptr, stop = nullptr;
    std::vector<cudaEvent_t> done;
    ~Events() {
      for (cudaEvent_t e : done)
        if (e) cudaEventDestroy(e);
      if (start) cudaEventDestroy(start);
      if (stop) cudaEventDestroy(stop);
    }
  } ev;
  ev.done.assign(S, nullptr);
  cudaEvent_t& start = ev.start;
  cudaEvent_t& stop = ev.stop;
  std::vector<cudaEvent_t>& done = ev.done;
  cuda_check(cudaEventCreate(&start), "event");
  cuda_check(cudaEventCreate(&stop), "event");
  for (auto& e : done) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  cuda_check(cudaEventRecord(start, st_), "event");
  for (int s = 0; s < S; ++s) cuda_check(cudaStreamWaitEvent(eng_[s]->stream(), start, 0), "wait");
  parallel_samples(S, threads_, device_, [&](int s) {
    Engine& e = *eng_[s];
    e.reset_state();
    e.record(false);
    e.record(true);
    for (int f = 0; f < frames; ++f) e.step();
    hdk_check_b(hdk_half_sqdist(n3, e.d_positions(), target_, loss_ + s, e.stream()), "loss");
    e.backward(nullptr, nullptr, nullptr, true, false, target_);
    e.record(false);
    cuda_check(cudaEventRecord(done[s], e.stream()), "event");
  });
  for (int s = 0; s < S; ++s) cuda_check(cudaStreamWaitEvent(st_, done[s], 0), "wait");
  hdk_check_b(hdk_batch_sum(S, ne, grads_, loss_, out_, st_), "batch sum");
  own_launches_ += S + 1;
  if (device_out)
    cuda_check(cudaMemcpyAsync(device_out, out_, (1 + static_cast<size_t>(ne)) * sizeof(double),
                               cudaMemcpyDeviceToDevice, st_),
               "device out");
  cuda_check(cudaEventRecord(stop, st_), "event");
  if (loss) cuda_check(cudaMemcpyAsync(loss, loss_, S * sizeof(double), cudaMemcpyDeviceToHost, st_), "loss out");
  if (grad_sum)
    cuda_check(cudaMemcpyAsync(grad_sum, out_ + 1, ne * sizeof(double), cudaMemcpyDeviceToHost, st_), "grad out");
  cuda_check(cudaStreamSynchronize(st_), "batch sync");
  float ms = 0;
  cuda_check(cudaEventElapsedTime(&ms, start, stop), "elapsed");
  last_ms = ms;
}

void Batch::evaluate_lockstep(int frames, double* loss, double* grad_sum, double* device_out) {
  Engine& e = *lock_;
  const int ne = scene_.mesh.ne;
  const hdk_segs& g = e.segs();
  e.reserve_frames(frames);
  struct Events {
    cudaEvent_t start = nullptr, stop = nullptr;
    ~Events() {
      if (start) cudaEventDestroy(start);
      if (stop) cudaEventDestroy(stop);
    }
  } ev;
  cuda_check(cudaEventCreate(&ev.start), "event");
  cuda_check(cudaEventCreate(&ev.stop), "event");
  cuda_check(cudaEventRecord(ev.start, st_), "event");
  e.reset_state();
  e.record(false);
  e.record(true);
  for (int f = 0; f < frames; ++f) e.step();
  hdk_check_b(hdk_seg_half_sqdist(&g, e.d_positions(), target_, loss_, st_), "loss");
  e.backward(nullptr, nullptr, nullptr, true, false, target_);  // L_s = 1/2 |q_T,s - q_target|^2 seeds
  e.record(false);
  hdk_check_b(hdk_seg_sum(&g, e.d_dl_de(), loss_, out_, st_), "batch sum");
  own_launches_ += 2;
  if (device_out)
    cuda_check(cudaMemcpyAsync(device_out, out_, (1 + static_cast<size_t>(ne)) * sizeof(double),
                               cudaMemcpyDeviceToDevice, st_), "device out");
  cuda_check(cudaEventRecord(ev.stop, st_), "event");
  if (loss) cuda_check(cudaMemcpyAsync(loss, loss_, samples_ * sizeof(double), cudaMemcpyDeviceToHost, st_), "loss out");
  if (grad_sum)
    cuda_check(cudaMemcpyAsync(grad_sum, out_ + 1, ne * sizeof(double), cudaMemcpyDeviceToHost, st_), "grad out");
  cuda_check(cudaStreamSynchronize(st_), "batch sync");
  float ms = 0;
  cuda_check(cudaEventElapsedTime(&ms, ev.start, ev.stop), "elapsed");
  last_ms = ms;
}

void Batch::set_young(const double* young, bool freeze_means) {
  const int ne = scene_.mesh.ne;
  if (lock_) {
    lock_->set_young(Vec(young, young + static_cast<size_t>(ne) * samples_), freeze_means);
    return;
  }
  parallel_samples(samples(), threads_, device_, [&](int s) {
    const Vec y(young + static_cast<size_t>(s) * ne, young + static_cast<size_t>(s + 1) * ne);
    eng_[s]->set_young(y, freeze_means);
  });
}

double Batch::time_solve(int reps, double* bytes) {
  return lock_ ? lock_->time_solve(reps, bytes) : eng_.front()->time_solve(reps, bytes);
}

long long Batch::solve_count() const {
  if (lock_) return lock_->solve_count * samples_;  // every lockstep solve streams all samples' factors
  long long k = 0;
  for (const auto& e : eng_) k += e->solve_count;
  return k;
}

double Batch::solve_bytes() const {
  if (lock_) {  // one sample's share of the block-diagonal stream
    const HostFactor& F = lock_->factor();
    return (16.0 * static_cast<double>(F.row_off.back()) + 96.0 * F.n) / samples_;
  }
  const HostFactor& F = eng_.front()->factor();
  return 16.0 * static_cast<double>(F.row_off.back()) + 96.0 * F.n;
}

long long Batch::kernel_launches() const {
  if (lock_) return own_launches_ + lock_->kernel_launches;
  long long k = own_launches_;
  for (const auto& e : eng_) k += e->kernel_launches;
  return k;
}

}  // namespace hdb
