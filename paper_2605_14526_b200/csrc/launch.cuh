// Kernel launch with programmatic dependent launch (PDL): consecutive kernels
// of the PD / adjoint loops are chained with programmatic edges, so a kernel
// is dispatched while its predecessor drains and waits at pdl_wait() (the
// start of every kernel here) for the predecessor's results — the launch gap
// between the ~10 kernels of one iteration is hidden.  Set HETERODYN_NO_PDL=1
// to launch plainly.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace hdk {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HETERODYN_NO_PDL");
    return !(e && std::atoi(e) != 0);
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// L2 residency hints.  The global solve streams ~340 MB per iteration
// through the 126 MB L2 (marked evict_first, solve.cu); the per-iteration
// working set the small kernels reuse every iteration (Anderson history,
// element differentials, element forces, iterates) is marked evict_last so
// it survives the stream.
__device__ __forceinline__ unsigned long long pol_keep() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_keep(const double* a, unsigned long long pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldg_keep(const double* a, unsigned long long pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_keep(double* a, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}

// In-graph timeline tracing (profiling).  Each translation unit owns a trace
// pointer (set through hdk_trace_install_<tu>, NULL = off); a traced kernel
// records, per kernel id, the earliest CTA start before and after its PDL
// wait and the latest CTA end (thread 0, globaltimer ns).
enum TraceId { kTrBapply, kTrGather, kTrRowdot, kTrZfold, kTrColtile, kTrDots, kTrMix,
               kTrTail0, kTrTail1, kTrTail2, kTrDotsA, kTrDotsB, kTrTail3, kTrTail4, kTrCount };  // tail stamps: AA tail entry, after fold, after solve

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Buffer layout: [0] epoch (bumped by hdk_trace_epoch before each traced
// body), then kTraceSlots epochs x kTrCount kernels x {pre-wait, start, end}.
constexpr int kTraceSlots = 16;
__device__ __forceinline__ unsigned long long* trace_rec(unsigned long long* buf, int id) {
  const unsigned long long ep = *reinterpret_cast<volatile unsigned long long*>(buf);
  return buf + 1 + 3 * ((ep % kTraceSlots) * kTrCount + id);
}
struct TraceScope {
  unsigned long long* rec;
  __device__ __forceinline__ TraceScope(unsigned long long* buf, int id) : rec(buf ? trace_rec(buf, id) : nullptr) {
    if (rec && threadIdx.x == 0) atomicMin(rec + 1, gtime());
  }
  __device__ __forceinline__ ~TraceScope() {
    if (rec && threadIdx.x == 0) atomicMax(rec + 2, gtime());
  }
};

// Point stamp (thread 0 of the calling CTA): latest time slot `id` was reached.
__device__ __forceinline__ void trace_stamp(unsigned long long* buf, int id) {
  if (buf && threadIdx.x == 0) atomicMax(trace_rec(buf, id) + 2, gtime());
}

}  // namespace hdk

// Per-TU trace pointer + its installer (extern "C" hdk_trace_install_<tu>).
#define HDK_TRACE_TU(tu)                                                        \
  namespace {                                                                    \
  __device__ unsigned long long* g_hdk_trace = nullptr;                          \
  }                                                                              \
  extern "C" HDK_API int hdk_trace_install_##tu(unsigned long long* buf) {       \
    return static_cast<int>(cudaMemcpyToSymbol(g_hdk_trace, &buf, sizeof(buf))); \
  }
// First statement of a traced kernel (replaces hdk::pdl_wait()).
#define HDK_TRACED_WAIT(id)                                                                \
  const unsigned long long hdk_trace_t0_ = g_hdk_trace ? hdk::gtime() : 0ULL;            \
  hdk::pdl_wait();                                                                         \
  hdk::TraceScope hdk_trace_scope_(g_hdk_trace, (id));                                     \
  if (hdk_trace_scope_.rec && threadIdx.x == 0) atomicMin(hdk_trace_scope_.rec, hdk_trace_t0_)
