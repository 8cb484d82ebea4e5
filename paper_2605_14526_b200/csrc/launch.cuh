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

}  // namespace hdk
